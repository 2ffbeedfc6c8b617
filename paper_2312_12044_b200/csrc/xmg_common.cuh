// xmg_common.cuh — shared device building blocks (included by xmg_step.cu
// inside its anonymous namespace): Philox4x64-10 and keys (ref:rng.py),
// entity codes and class masks (ref:core.py), cp.async staging, the per-env
// views of a grid, the MOVE / PICK_UP rules and goals (ref:rules.py,
// ref:goals.py) and the egocentric observation (ref:observation.py).

// ------------------------------------------------------------------ Philox
// ref:rng.py:23-32
constexpr uint64_t kM0 = 0xD2E7470EE14C6C93ULL;
constexpr uint64_t kM1 = 0xCA5A826395121157ULL;
constexpr uint64_t kW0 = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kW1 = 0xBB67AE8584CAA73BULL;
constexpr uint64_t kDomDraw = 1, kDomSplit = 2, kDomSeed = 4;

struct Words4 {
  uint64_t w0, w1, w2, w3;
};

// Philox4x64-10, ref:rng.py:42-57.  __umul64hi gives the high half of the
// 64x64 product the reference builds from 32-bit limbs (rng.py:60-71).
template <int UNROLL = 10>
__device__ __forceinline__ Words4 philox(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3, uint64_t k0,
                                         uint64_t k1) {
#pragma unroll UNROLL
  for (int r = 0; r < 10; ++r) {
    const uint64_t hi0 = __umul64hi(kM0, c0), lo0 = kM0 * c0;
    const uint64_t hi1 = __umul64hi(kM1, c2), lo1 = kM1 * c2;
    const uint64_t n0 = hi1 ^ c1 ^ k0;
    const uint64_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += kW0;
    k1 += kW1;
  }
  return {c0, c1, c2, c3};
}

void philox_host(const uint64_t ctr[4], uint64_t k0, uint64_t k1, uint64_t out[4]) {
  uint64_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  for (int r = 0; r < 10; ++r) {
    const unsigned __int128 p0 = (unsigned __int128)kM0 * c0;
    const unsigned __int128 p1 = (unsigned __int128)kM1 * c2;
    const uint64_t n0 = (uint64_t)(p1 >> 64) ^ c1 ^ k0;
    const uint64_t n2 = (uint64_t)(p0 >> 64) ^ c3 ^ k1;
    c1 = (uint64_t)p1;
    c3 = (uint64_t)p0;
    c0 = n0;
    c2 = n2;
    k0 += kW0;
    k1 += kW1;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// ------------------------------------------------------------------ codes
// ref:core.py:17-70; ref:layouts.py:39-42
constexpr int kFloor = 3, kWall = 4, kBall = 5, kGoal = 8, kKey = 9, kLocked = 10, kClosed = 11, kOpen = 12;
constexpr uint8_t kFloorCode = 57, kWallCode = 72, kGreenGoal = 132;
__constant__ uint8_t cGenColors[10] = {3, 4, 5, 6, 7, 8, 10, 11, 12, 13};
// tile-class bitmasks over the tile nibble (ref:core.py:53-59, ref:observation.py:21)
constexpr uint32_t kWalkable = (1u << kFloor) | (1u << kGoal) | (1u << kOpen);
constexpr uint32_t kPickable = (1u << 5) | (1u << 6) | (1u << 7) | (1u << 9) | (1u << 13) | (1u << 14);
constexpr uint32_t kOpaque = (1u << kWall) | (1u << kClosed) | (1u << kLocked);
// trigger gates as event bitmasks (ref:rules.py:60-72, ref:goals.py:51-66)
__constant__ uint8_t cRuleGate[12] = {0, 0x2, 0x7, 0x4, 0x4, 0x4, 0x4, 0x4, 0x7, 0x7, 0x7, 0x7};
__constant__ uint8_t cGoalGate[15] = {0, 0x2, 0x7, 0x7, 0x4, 0x7, 0x4, 0x4, 0x4, 0x4, 0x4, 0x7, 0x7, 0x7, 0x7};

// direction deltas (ref:core.py:122)
__device__ __forceinline__ int dir_dr(int d) { return d == 0 ? -1 : (d == 2 ? 1 : 0); }
__device__ __forceinline__ int dir_dc(int d) { return d == 1 ? 1 : (d == 3 ? -1 : 0); }
// NEAR_OFFSETS = up, left, right, down (ref:rules.py:76)
__device__ __forceinline__ int near_dr(int k) { return k == 0 ? -1 : (k == 3 ? 1 : 0); }
__device__ __forceinline__ int near_dc(int k) { return k == 1 ? -1 : (k == 2 ? 1 : 0); }

#ifndef XMG_THREADS
#define XMG_THREADS 64  // 64-env CTAs: C3 78.2 -> 76.9, C4 54.1 -> 51.5 us/step vs 128 (256: slower)
#endif
constexpr int kThreads = XMG_THREADS;  // envs per step_main CTA
constexpr int kStatEnvs = 128;         // envs per episode-statistics slot (include/xmg.h xmg_out.stats)
constexpr int kRowHeader = 4;  // task row: goal, counts, MOVE slot mask, PICK_UP slot mask
constexpr int kMaxDynSmem = 227 * 1024 - 1024;  // leave room for the static shared desc copy
constexpr int kWarps = kThreads / 32;
#ifdef XMG_TRACE
// debug builds: per-warp phase timestamps of step_rare (globaltimer, ns);
// columns 0..7 step_rare phases, 8..23 the first warp_build of the warp
__device__ unsigned long long g_trace[1 << 16][24];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define XMG_TR(gw, k, v) \
  if ((threadIdx.x & 31) == 0 && (gw) < (1 << 16)) g_trace[gw][k] = (v)
#define XMG_TRB(k)                                                                                  \
  {                                                                                                 \
    const int gw_ = blockIdx.x * kWarps + (threadIdx.x >> 5);                                       \
    if ((threadIdx.x & 31) == 0 && gw_ < (1 << 16) && g_trace[gw_][8 + (k)] == 0) g_trace[gw_][8 + (k)] = gtime(); \
  }
#else
#define XMG_TR(gw, k, v)
#define XMG_TRB(k)
#endif
#ifndef XMG_MINB
#define XMG_MINB (1024 / XMG_THREADS)  // min resident CTAs per SM the register allocation targets (64 registers; measured best at C3)
#endif
#ifndef XMG_MINB_RARE
#define XMG_MINB_RARE 6  // step_rare: <= 80 registers, so the next step's kernels fit beside it
#endif
#ifndef XMG_RARE
#define XMG_RARE __forceinline__  // rare paths (reset, PUT_DOWN, occlusion) inlined: measured faster
#endif

__host__ __device__ inline int round16(int x) { return (x + 15) & ~15; }

// chunk capacity needed for the (MOVE-extended) window: span = v*W + v bytes
inline int needed_chunks(int W, int V) { return (V * W + V + 30) / 16; }

// ------------------------------------------------------- async copies
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async16_hint(void* smem_dst, const void* gmem_src, uint64_t pol) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem_src), "l"(pol)
               : "memory");
}
// the same with the shared-memory address already converted (one
// generic->shared conversion per buffer instead of one per chunk)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16_s(uint32_t s, const void* gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async16_hint_s(uint32_t s, const void* gmem_src, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem_src), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------- debug checks
// XMG_CHECKS builds (tests/test_parity_gpu.py::test_checked_build_parity)
// trap on any index outside the buffer it addresses: the stand-in for
// compute-sanitizer, which this pool does not run.
#ifdef XMG_CHECKS
#define XMG_ASSERT(c) \
  do {                \
    if (!(c)) __trap(); \
  } while (0)
#else
#define XMG_ASSERT(c) \
  do {                \
  } while (0)
#endif

// ------------------------------------------------------- per-thread view
// The bytes of one env's grid staged in shared memory: stage[k] mirrors grid
// flat index sbase + k for flat indices in [slo, shi); everything else falls
// through to global memory.
struct View {
  uint8_t* g;      // env grid in global memory
  uint8_t* stage;  // per-thread shared stage (nullptr when unused)
  int sbase, slo, shi;

  __device__ __forceinline__ uint8_t rd(int f) const {
    XMG_ASSERT(f >= 0);
    return (f >= slo && f < shi) ? stage[f - sbase] : g[f];
  }
  __device__ __forceinline__ void wr(int f, uint8_t v) const {
    XMG_ASSERT(f >= 0);
    g[f] = v;
    if (f >= slo && f < shi) stage[f - sbase] = v;
  }
};

// Bounding box of the view window for pose (r, c, d), extended by `ext`
// cells ahead and `back` cells behind (ref:vecenv.py:77-92 /
// ref:observation.py:28-43), clipped.
__device__ __forceinline__ void window_span(int r, int c, int d, int ext, int back, int H, int W, int V, int& lo,
                                            int& hi) {
  const int h = V / 2, far = V - 1 + ext;
  // select-based (lanes facing different ways stay converged)
  int r0 = d == 0 ? r - far : d == 2 ? r - back : r - h;
  int r1 = d == 0 ? r + back : d == 2 ? r + far : r + h;
  int c0 = d == 1 ? c - back : d == 3 ? c - far : c - h;
  int c1 = d == 1 ? c + far : d == 3 ? c + back : c + h;
  r0 = max(r0, 0); c0 = max(c0, 0); r1 = min(r1, H - 1); c1 = min(c1, W - 1);
  lo = r0 * W + c0;
  hi = r1 * W + c1 + 1;
}

// The staged window of step_main: it always covers every cell the step reads
// (the view of the post-action pose, one cell further ahead for MOVE and one
// behind for PICK_UP, whose agent-relative rules see all four neighbours),
// so reads need no range check; writes go through to the grid in HBM.
struct WView : View {
  __device__ __forceinline__ uint8_t rd(int f) const {
    XMG_ASSERT(f >= slo && f < shi);  // the invariant that makes the unchecked read safe
    return stage[f - sbase];
  }
  __device__ __forceinline__ void wr(int f, uint8_t v) const {
    XMG_ASSERT(f >= slo && f < shi);
    View::wr(f, v);
  }
};

// four signed bytes packed into a word (byte k = v_k), and the replication
// factor that copies a VV-bit group into all VV row groups of a VV*VV mask
__host__ __device__ constexpr uint32_t sbytes4(int a, int b, int c, int d) {
  return (uint32_t)(a & 0xff) | ((uint32_t)(b & 0xff) << 8) | ((uint32_t)(c & 0xff) << 16) |
         ((uint32_t)(d & 0xff) << 24);
}
// byte (sel & 7) of k, sign-extended: prmt with the sign-replicate bit set
// in the upper three selectors (sel = d * 0x1111 + 0x8880 picks byte d).  PTX
// directly: the __byte_perm intrinsic takes 3-bit selectors only.
__device__ __forceinline__ int sbyte_of(uint32_t k, uint32_t sel) {
  uint32_t v;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(v) : "r"(k), "r"(sel));
  return (int)v;
}
__host__ __device__ constexpr uint32_t rep_groups(int vv) {
  uint32_t m = 0;
  for (int i = 0; i < vv; ++i) m |= 1u << (i * vv);
  return m;
}

// Stage grid bytes [lo, hi) of this thread's env with 16-byte cp.async
// chunks (aligned on the global address; the grid buffer is padded).
template <int MAXCH>
__device__ __forceinline__ void stage_issue(View& vw, int lo, int hi, int HW, const uint64_t* pol = nullptr) {
  if constexpr (MAXCH == 0) {
    vw.slo = vw.shi = vw.sbase = 0;
  } else {
    const uintptr_t gb = reinterpret_cast<uintptr_t>(vw.g);
    const uintptr_t a0 = (gb + lo) & ~uintptr_t(15);
    const int nch = (int)((gb + hi - a0 + 15) >> 4);
    vw.sbase = (int)(a0 - gb);
    vw.slo = max(vw.sbase, 0);
    vw.shi = min(vw.sbase + 16 * nch, HW);
    const uint32_t sb = smem_u32(vw.stage);
#pragma unroll
    for (int k = 0; k < MAXCH; ++k)
      if (k < nch) {
        if (pol) cp_async16_hint_s(sb + 16 * k, reinterpret_cast<const void*>(a0 + 16 * k), *pol);
        else cp_async16_s(sb + 16 * k, reinterpret_cast<const void*>(a0 + 16 * k));
      }
  }
}

// ------------------------------------------------------- rules and goals
// ref:rules.py:147-217 (scalar) / ref:vecenv.py:368-433 (batched).  Slots in
// stored order, each sees earlier rewrites.
//
// MOVE and PICK_UP events gate only agent-relative rules (AGENT_HOLD,
// AGENT_NEAR, AGENT_NEAR_{UP,RIGHT,DOWN,LEFT}) and agent-relative goals, so
// they are resolved per lane from the staged window.  Every grid-wide
// predicate (TILE_NEAR* rules, TILE_* goals) is gated on PUT_DOWN only
// (ref:rules.py:60-72, ref:goals.py:51-66): PUT_DOWN events are queued and
// resolved by step_rare (warp_put_env).
// The agent's four neighbour cells in NEAR_OFFSETS order (up, left, right,
// down; ref:rules.py:76), 0x100 when off the grid, plus their flat indices.
struct Nbrs {
  int code[4];
  int flat[4];
};

// A grid staged whole in shared memory (the rollout kernel): no range checks.
struct SView {
  uint8_t* stage;
#ifdef XMG_CHECKS
  int hw = 1 << 30;
#endif
  __device__ __forceinline__ uint8_t rd(int f) const {
#ifdef XMG_CHECKS
    XMG_ASSERT(f >= 0 && f < hw);
#endif
    return stage[f];
  }
  __device__ __forceinline__ void wr(int f, uint8_t v) const {
#ifdef XMG_CHECKS
    XMG_ASSERT(f >= 0 && f < hw);
#endif
    stage[f] = v;
  }
};

template <class VW>
__device__ __forceinline__ Nbrs load_nbrs(const VW& vw, int H, int W, int ar, int ac) {
  Nbrs nb;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = ar + near_dr(k), c = ac + near_dc(k);
    const bool in = r >= 0 && r < H && c >= 0 && c < W;
    nb.flat[k] = r * W + c;
    nb.code[k] = in ? (int)vw.rd(nb.flat[k]) : 0x100;
  }
  return nb;
}

// NEAR_OFFSETS slot of the directional offsets up, right, down, left
// (ref:rules.py:80-89, ref:goals.py:70-79)
__device__ __forceinline__ int dir_slot(int d) { return d == 0 ? 0 : d == 1 ? 2 : d == 2 ? 3 : 1; }

// Rules gated on MOVE / PICK_UP (only the slots in `slots`, stored order).
// Select-based, so lanes holding different rule kinds stay converged.
template <class VW>
__device__ XMG_RARE int agent_rules(VW vw, Nbrs& nb, const uint32_t* rules, uint32_t slots, int pocket) {
  for (; slots; slots &= slots - 1) {
    const uint32_t rw = rules[__ffs(slots) - 1];
    const int kind = rw & 0xff, a = (rw >> 8) & 0xff, out = rw >> 24;
    // AGENT_HOLD
    pocket = (kind == 1 && pocket == a) ? ((out >> 4) == kFloor ? 0 : out) : pocket;
    // AGENT_NEAR: first neighbour holding a (slots up, left, right, down);
    // AGENT_NEAR_{UP,RIGHT,DOWN,LEFT}: the one slot of that direction
    const uint32_t m = (uint32_t)(nb.code[0] == a) | ((uint32_t)(nb.code[1] == a) << 1) |
                       ((uint32_t)(nb.code[2] == a) << 2) | ((uint32_t)(nb.code[3] == a) << 3);
    const uint32_t allow = (rw >> 16) & 0xFu;  // the table's neighbour-slot mask (0 for AGENT_HOLD)
    const uint32_t hit = m & allow;
    if (hit) {
      const int k = __ffs(hit) - 1;
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (t == k) {
          nb.code[t] = out;
          vw.wr(nb.flat[t], (uint8_t)out);
        }
    }
  }
  return pocket;
}

// Agent-relative goals (ref:goals.py:144-161); the TILE_* kinds never pass the
// gate of a MOVE / PICK_UP event.
__device__ __forceinline__ bool agent_goal(const Nbrs& nb, int own, uint32_t goal, int ev, int ar, int ac,
                                           int pocket) {
  const int kind = goal & 0xff, a1 = (goal >> 8) & 0xff, a2 = (goal >> 16) & 0xff;
  if (kind == 0 || kind > 14 || !((cGoalGate[kind] >> ev) & 1)) return false;
  // select-based (no per-kind branches)
  const uint32_t m = (uint32_t)(nb.code[0] == a1) | ((uint32_t)(nb.code[1] == a1) << 1) |
                     ((uint32_t)(nb.code[2] == a1) << 2) | ((uint32_t)(nb.code[3] == a1) << 3);
  const uint32_t allow = kind == 3 ? 0xFu : (kind >= 11 && kind <= 14) ? (0x2841u >> (4 * (kind - 11))) & 0xFu : 0u;
  return (m & allow) != 0 || (kind == 1 && pocket == a1) || (kind == 2 && own == a1) ||
         (kind == 5 && ar == a1 && ac == a2);
}

// ------------------------------------------------------- observation
// See-through view (ref:vecenv.py:481-500): view cell (i, j) is world
// (r0 + i*dri + j*drj, c0 + i*dci + j*dcj), an affine map per facing;
// off-grid cells read END_OF_MAP (0, 0).  Output pairs (tile, color).
template <int VV>
__device__ __forceinline__ void obs_see(const uint8_t* stage, int sbase, uint8_t* dst, int r, int c, int d, int H,
                                        int W, int Vrt) {
  const int V = VV ? VV : Vrt;
  const int h = V / 2;
  // origin (view cell (0, 0)) and the world steps of i (rows) and j
  // (columns).  The j step is (-dci, dri): the view's columns run to the
  // agent's right.
  int r0, c0, dri, dci;
  if constexpr (VV != 0) {
    // per-facing constants as signed bytes (facing d in byte d), picked with
    // one sign-extending byte permute each (lanes facing different ways stay
    // converged, no select chains)
    constexpr int F = VV - 1, HH = VV / 2;
    constexpr uint32_t kR0 = sbytes4(-F, -HH, F, HH), kC0 = sbytes4(-HH, F, HH, -F);
    constexpr uint32_t kRI = sbytes4(1, 0, -1, 0), kCI = sbytes4(0, -1, 0, 1);
    const uint32_t sel = (uint32_t)d * 0x1111u + 0x8880u;
    r0 = r + sbyte_of(kR0, sel);
    c0 = c + sbyte_of(kC0, sel);
    dri = sbyte_of(kRI, sel);
    dci = sbyte_of(kCI, sel);
  } else {
    const bool d0 = d == 0, d1 = d == 1, d2 = d == 2;
    r0 = d0 ? r - (V - 1) : d2 ? r + (V - 1) : d1 ? r - h : r + h;
    c0 = d0 ? c - h : d2 ? c + h : d1 ? c + (V - 1) : c - (V - 1);
    dri = d0 ? 1 : d2 ? -1 : 0;
    dci = d1 ? -1 : (d0 || d2) ? 0 : 1;
  }
  const int drj = -dci, dcj = dri;
  // the facing makes i move along one world axis and j along the other
  // (i along rows iff the facing is vertical): validity is a product of a
  // range [lo, hi) over i and one over j
  const bool vert = (d & 1) == 0;
  auto range = [V](int b, int st, int lim, int& lo, int& hi) {  // t in [0, V) with 0 <= b + t*st < lim
    lo = st > 0 ? -b : b - lim + 1;
    hi = st > 0 ? lim - b : b + 1;
    lo = max(lo, 0);
    hi = min(hi, V);
  };
  int loi, hii, loj, hij;
  range(vert ? r0 : c0, vert ? dri : dci, vert ? H : W, loi, hii);
  range(vert ? c0 : r0, vert ? dcj : drj, vert ? W : H, loj, hij);
  const uint32_t mi = hii > loi ? ((1u << hii) - 1u) & ~((1u << loi) - 1u) : 0u;
  const uint32_t mj = hij > loj ? ((1u << hij) - 1u) & ~((1u << loj) - 1u) : 0u;
  const int di = dri * W + dci, dj = drj * W + dcj;  // flat steps
  const uint8_t* p0 = stage - sbase + (r0 * W + c0);
  // (tile, color) byte pairs as 16-bit values; written as one u16 plus
  // (V*V - 1) / 2 u32 words (the record is 2-byte aligned: an odd-offset
  // record leads with its u16, an even one ends with it)
  const bool odd = (reinterpret_cast<uintptr_t>(dst) & 2) != 0;
  if constexpr (VV != 0) {
    constexpr int NC = VV * VV;
    uint32_t cd[NC + 3];  // entity codes, view cell order (+ zero pads to a multiple of 4)
    int jo[VV];           // column offsets, once per view (not per cell)
#pragma unroll
    for (int j = 0; j < VV; ++j) jo[j] = j * dj;
    static_assert(VV * VV <= 32, "the cell mask is one 32-bit word");
    // validity of every view cell: bit i*VV + j = mi bit i and mj bit j —
    // mj copied into every row group by one multiply, the rows [loi, hii) as
    // one bit range
    constexpr uint32_t kRep = rep_groups(VV);
    const uint32_t rows = hii > loi ? ((1u << (VV * hii)) - 1u) & ~((1u << (VV * loi)) - 1u) : 0u;
    const uint32_t m25 = rows & (mj * kRep);
    (void)mi;
    const uint8_t* pi = p0;
#pragma unroll
    for (int i = 0; i < VV; ++i) {
#pragma unroll
      for (int j = 0; j < VV; ++j) {
        uint32_t code = 0;
        if ((m25 >> (i * VV + j)) & 1u) code = pi[jo[j]];
        cd[i * VV + j] = code;
      }
      pi += di;
    }
#pragma unroll
    for (int k = NC; k < NC + 3; ++k) cd[k] = 0;
    // four cells -> two (tile, color, tile, color) words: pack the codes
    // (3 byte_perms), split the nibbles (3 ALU ops), interleave (2 byte_perms)
    uint32_t ev[(NC + 3) / 2];  // even-aligned words: cells (2k, 2k+1)
#pragma unroll
    for (int q = 0; q < (NC + 3) / 4; ++q) {
      const uint32_t x = __byte_perm(__byte_perm(cd[4 * q], cd[4 * q + 1], 0x0040),
                                     __byte_perm(cd[4 * q + 2], cd[4 * q + 3], 0x0040), 0x5410);
      const uint32_t hi = (x >> 4) & 0x0F0F0F0Fu, lo = x & 0x0F0F0F0Fu;
      ev[2 * q] = __byte_perm(hi, lo, 0x5140);
      ev[2 * q + 1] = __byte_perm(hi, lo, 0x7362);
    }
    // an odd-offset record leads with cell 0 as a u16, then words of cells
    // (2k+1, 2k+2) = the even words shifted by one cell; an even one ends
    // with cell NC-1 as a u16
    *reinterpret_cast<uint16_t*>(dst + (odd ? 0 : 2 * (NC - 1))) =
        (uint16_t)(odd ? ev[0] : ev[(NC - 1) / 2]);
    uint32_t* d32 = reinterpret_cast<uint32_t*>(dst + (odd ? 2 : 0));
    const uint32_t sh = odd ? 16u : 0u;  // a funnel shift by 0 is the word itself
#pragma unroll
    for (int k = 0; k < (NC - 1) / 2; ++k) d32[k] = __funnelshift_r(ev[k], ev[k + 1], sh);
  } else {
    uint16_t* o = reinterpret_cast<uint16_t*>(dst);
    for (int i = 0; i < V; ++i)
      for (int j = 0; j < V; ++j) {
        uint32_t code = 0;
        if (((mi >> i) & (mj >> j)) & 1) code = p0[i * di + j * dj];
        o[i * V + j] = (uint16_t)(((code * 0x1001u) >> 4) & 0x0F0Fu);
      }
  }
}

// exact-integer line of sight, ref:observation.py:46-87
__device__ bool seg_crosses_cell(int p0r, int p0c, int dr, int dc, int cr, int cc) {
  int lo_n = 0, lo_d = 1, hi_n = 1, hi_d = 1;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int p0 = k ? p0c : p0r, d = k ? dc : dr, low = 2 * (k ? cc : cr), high = low + 2;
    if (d == 0) {
      if (!(low < p0 && p0 < high)) return false;
      continue;
    }
    const int a = low - p0, b = high - p0;
    int ln, ld, hn, hd;
    if (d > 0) { ln = a; ld = d; hn = b; hd = d; } else { ln = -b; ld = -d; hn = -a; hd = -d; }
    if (ln * lo_d > lo_n * ld) { lo_n = ln; lo_d = ld; }
    if (hn * hi_d < hi_n * hd) { hi_n = hn; hi_d = hd; }
  }
  return lo_n * hi_d < hi_n * lo_d;
}

__device__ __noinline__ bool cell_visible_p(const uint8_t* stage, int sbase, int slo, int shi, const uint8_t* g, int W,
                                            int r0, int c0, int r1, int c1);

__device__ __forceinline__ bool cell_visible(const View& vw, int W, int r0, int c0, int r1, int c1) {
  return cell_visible_p(vw.stage, vw.sbase, vw.slo, vw.shi, vw.g, W, r0, c0, r1, c1);
}

__device__ __noinline__ bool cell_visible_p(const uint8_t* stage, int sbase, int slo, int shi, const uint8_t* g, int W,
                                            int r0, int c0, int r1, int c1) {
  View vw;
  vw.stage = const_cast<uint8_t*>(stage);
  vw.g = const_cast<uint8_t*>(g);
  vw.sbase = sbase;
  vw.slo = slo;
  vw.shi = shi;
  if (r0 == r1 && c0 == c1) return true;
  const int p0r = 2 * r0 + 1, p0c = 2 * c0 + 1, dr = 2 * (r1 - r0), dc = 2 * (c1 - c0);
  for (int rr = min(r0, r1); rr <= max(r0, r1); ++rr)
    for (int cc = min(c0, c1); cc <= max(c0, c1); ++cc) {
      if ((rr == r0 && cc == c0) || (rr == r1 && cc == c1)) continue;
      if (!((kOpaque >> (vw.rd(rr * W + cc) >> 4)) & 1)) continue;
      if (seg_crosses_cell(p0r, p0c, dr, dc, rr, cc)) return false;
    }
  return true;
}

// Occluded view (see_through_walls=False), ref:observation.py:90-110.
#ifndef XMG_OCC_INLINE
#define XMG_OCC_INLINE XMG_RARE
#endif
__device__ XMG_OCC_INLINE void obs_occluded(View vw, uint8_t* dst, int r, int c, int d, int H, int W, int V) {
  const int h = V / 2;
  const int fr = dir_dr(d), fc = dir_dc(d);
  const int rr = fc, rc = -fr;  // right-hand vector (ref:observation.py:25)
  uint16_t* o = reinterpret_cast<uint16_t*>(dst);
  for (int i = 0; i < V; ++i) {
    const int ahead = V - 1 - i;
    for (int j = 0; j < V; ++j) {
      const int lat = j - h;
      const int wr = r + ahead * fr + lat * rr, wc = c + ahead * fc + lat * rc;
      uint16_t v = 0;
      if (wr >= 0 && wr < H && wc >= 0 && wc < W) {
        if (!cell_visible(vw, W, r, c, wr, wc)) {
          v = 1 | (1 << 8);  // (UNSEEN, UNSEEN)
        } else {
          const int code = vw.rd(wr * W + wc);
          v = (uint16_t)((code >> 4) | ((code & 15) << 8));
        }
      }
      o[i * V + j] = v;
    }
  }
}
