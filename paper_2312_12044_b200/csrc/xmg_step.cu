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
//  * step_main — one thread per env, 128 envs per CTA: one 16-byte state word
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
//  * sprite_kernel / image_kernel (xmg_render.cuh) — 224x224 observation images.
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
// trigger gates as event bitmasks (ref:rules.py:60-72, ref:goals.py:268-283)
__constant__ uint8_t cRuleGate[12] = {0, 0x2, 0x7, 0x4, 0x4, 0x4, 0x4, 0x4, 0x7, 0x7, 0x7, 0x7};
__constant__ uint8_t cGoalGate[15] = {0, 0x2, 0x7, 0x7, 0x4, 0x7, 0x4, 0x4, 0x4, 0x4, 0x4, 0x7, 0x7, 0x7, 0x7};

// direction deltas (ref:core.py:272)
__device__ __forceinline__ int dir_dr(int d) { return d == 0 ? -1 : (d == 2 ? 1 : 0); }
__device__ __forceinline__ int dir_dc(int d) { return d == 1 ? 1 : (d == 3 ? -1 : 0); }
// NEAR_OFFSETS = up, left, right, down (ref:rules.py:76)
__device__ __forceinline__ int near_dr(int k) { return k == 0 ? -1 : (k == 3 ? 1 : 0); }
__device__ __forceinline__ int near_dc(int k) { return k == 1 ? -1 : (k == 2 ? 1 : 0); }

constexpr int kThreads = 128;  // envs per CTA
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
#define XMG_MINB 8  // min resident CTAs per SM the register allocation targets (64 registers; measured best at C3)
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

// Stage grid bytes [lo, hi) of this thread's env with 16-byte cp.async
// chunks (aligned on the global address; the grid buffer is padded).
template <int MAXCH>
__device__ __forceinline__ void stage_issue(View& vw, int lo, int hi, int HW) {
  if constexpr (MAXCH == 0) {
    vw.slo = vw.shi = vw.sbase = 0;
  } else {
    const uintptr_t gb = reinterpret_cast<uintptr_t>(vw.g);
    const uintptr_t a0 = (gb + lo) & ~uintptr_t(15);
    const int nch = (int)((gb + hi - a0 + 15) >> 4);
    vw.sbase = (int)(a0 - gb);
    vw.slo = max(vw.sbase, 0);
    vw.shi = min(vw.sbase + 16 * nch, HW);
#pragma unroll
    for (int k = 0; k < MAXCH; ++k)
      if (k < nch) cp_async16(vw.stage + 16 * k, reinterpret_cast<const void*>(a0 + 16 * k));
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
// (ref:rules.py:60-72, ref:goals.py:268-283): PUT_DOWN events are queued and
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
// (ref:rules.py:80-89, ref:goals.py:287-296)
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

// Agent-relative goals (ref:goals.py:361-378); the TILE_* kinds never pass the
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
  // (columns), select-based (lanes facing different ways stay converged)
  const bool d0 = d == 0, d1 = d == 1, d2 = d == 2;
  const int r0 = d0 ? r - (V - 1) : d2 ? r + (V - 1) : d1 ? r - h : r + h;
  const int c0 = d0 ? c - h : d2 ? c + h : d1 ? c + (V - 1) : c - (V - 1);
  const int dri = d0 ? 1 : d2 ? -1 : 0, dci = d1 ? -1 : (d0 || d2) ? 0 : 1;
  const int drj = d1 ? 1 : (d0 || d2) ? 0 : -1, dcj = d0 ? 1 : d2 ? -1 : 0;
  // the facing makes i move along one world axis and j along the other:
  // validity is a product of a bit range over i and one over j
  auto range_mask = [V](int b, int st, int lim) {  // t in [0, V) with 0 <= b + t*st < lim
    int lo = st > 0 ? -b : b - lim + 1, hi = st > 0 ? lim - b : b + 1;
    lo = max(lo, 0);
    hi = min(hi, V);
    return hi > lo ? ((1u << hi) - 1u) & ~((1u << lo) - 1u) : 0u;
  };
  const uint32_t mi = dri ? range_mask(r0, dri, H) : range_mask(c0, dci, W);
  const uint32_t mj = drj ? range_mask(r0, drj, H) : range_mask(c0, dcj, W);
  const int di = dri * W + dci, dj = drj * W + dcj;  // flat steps
  const uint8_t* p0 = stage - sbase + (r0 * W + c0);
  // (tile, color) byte pairs as 16-bit values; written as one u16 plus
  // (V*V - 1) / 2 u32 words (the record is 2-byte aligned: an odd-offset
  // record leads with its u16, an even one ends with it)
  const bool odd = (reinterpret_cast<uintptr_t>(dst) & 2) != 0;
  if constexpr (VV != 0) {
    constexpr int NC = VV * VV;
    uint32_t cd[NC + 1];  // entity codes, view cell order (+ a zero pad)
    int jo[VV];           // column offsets, once per view (not per cell)
#pragma unroll
    for (int j = 0; j < VV; ++j) jo[j] = j * dj;
    static_assert(VV * VV <= 32, "the cell mask is one 32-bit word");
    uint32_t m25 = 0;  // validity of every view cell: bit i*VV + j = mi bit i and mj bit j
#pragma unroll
    for (int i = 0; i < VV; ++i) m25 |= (((mi >> i) & 1u) ? mj : 0u) << (i * VV);
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
    cd[NC] = 0;
    // two cells -> one (tile, color, tile, color) word: pack the codes, split
    // nibbles, interleave (3 byte_perms + 3 ALU ops per pair)
    auto pair = [](uint32_t a, uint32_t b) {
      const uint32_t x = __byte_perm(a, b, 0x0040);
      return __byte_perm((x >> 4) & 0x0F0Fu, x & 0x0F0Fu, 0x5140);
    };
    uint32_t ev[(NC + 1) / 2];  // even-aligned words: cells (2k, 2k+1)
#pragma unroll
    for (int k = 0; k < (NC + 1) / 2; ++k) ev[k] = pair(cd[2 * k], cd[2 * k + 1]);
    // an odd-offset record leads with cell 0 as a u16, then words of cells
    // (2k+1, 2k+2) = the even words shifted by one cell; an even one ends
    // with cell NC-1 as a u16
    *reinterpret_cast<uint16_t*>(dst + (odd ? 0 : 2 * (NC - 1))) =
        (uint16_t)(odd ? ev[0] : ev[(NC - 1) / 2]);
    uint32_t* d32 = reinterpret_cast<uint32_t*>(dst + (odd ? 2 : 0));
#pragma unroll
    for (int k = 0; k < (NC - 1) / 2; ++k) d32[k] = odd ? __funnelshift_r(ev[k], ev[k + 1], 16) : ev[k];
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
__device__ XMG_RARE void obs_occluded(View vw, uint8_t* dst, int r, int c, int d, int H, int W, int V) {
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

// Row-major floor cells of the scratch grid into fc[]; returns their count
// (the free list of ref:core.py:322-325, built with ballots).
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

// Warp radix-select over the draw words (ref:core.py:328-333,
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
  for (int b = 31; b >= 0 && cc > 1; --b) {
    uint32_t z = 0;
#pragma unroll
    for (int j = 0; j < 4 * KR; ++j) z |= ((~hi[j] >> b) & 1u) << j;
    z &= c;
    const int zeros = (int)__reduce_add_sync(0xffffffffu, (unsigned)__popc(z));
    if (tt < zeros) {
      c = z;
      cc = zeros;
    } else {
      c &= ~z;
      tt -= zeros;
      cc -= zeros;
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
// spawn_base) (ref:scenarios.py:281-288), via warp_select: the element of
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
    const int fs = select_rank(ws.wd, lane, F, valid, total, spawn_base + (int)(spawn_word % (uint64_t)tail));
    if (lane == 0) reinterpret_cast<int*>(ws.misc + 32)[0] = ws.fc[fs];
  }
  __syncwarp();
}

// Every key a trial reset consumes, derived from the episode key ek:
// ref:vecenv.py:224-227 (ks = split(ek, 0), next state key st = split(ek, 1))
// and ref:scenarios.py:293,344,363,376 (k0, k1, k2 = split(ks, 3)); see
// warp_trial_keys.
struct TrialKeys {
  uint64_t st_hi, st_lo, k0h, k0l, k1h, k1l, k2h, k2l, task_word;
};

__device__ __noinline__ void derive_trial_keys(uint64_t ek_hi, uint64_t ek_lo, bool resample, TrialKeys* out) {
  TrialKeys k;
  const Words4 ks = philox<2>(0, 0, kDomSplit, 0, ek_hi, ek_lo);
  const Words4 st = philox<2>(1, 0, kDomSplit, 0, ek_hi, ek_lo);
  k.st_hi = st.w0;
  k.st_lo = st.w1;
  uint64_t sub[6];
#pragma unroll 1
  for (int i = 0; i < 3; ++i) {
    const Words4 w = philox<2>((uint64_t)i, 0, kDomSplit, 0, ks.w0, ks.w1);
    sub[2 * i] = w.w0;
    sub[2 * i + 1] = w.w1;
  }
  k.k0h = sub[0]; k.k0l = sub[1];
  k.k1h = sub[2]; k.k1l = sub[3];
  k.k2h = sub[4]; k.k2l = sub[5];
  k.task_word = 0;
  if (resample) {
    // extension (not in the reference): a fresh task per trial, drawn as
    // Benchmark.sample_ruleset(split(ek, 2)) = rows[word0 % M] (ref:benchio.py:57-58)
    const Words4 tk = philox<2>(2, 0, kDomSplit, 0, ek_hi, ek_lo);
    k.task_word = philox<2>(0, 0, kDomDraw, 0, tk.w0, tk.w1).w0;
  }
  *out = k;
}

// Rebuild one env's trial with the scenario builders ref:scenarios.py:291-412
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
  // ref:scenarios.py:361-370; EmptyRandom: none)
  int nobj = 0, obj_lane = 0;
  if (sc == XMG_SCENARIO_XLAND) {
    nobj = (int)((row[1] >> 8) & 0xff);
    if (lane < nobj) obj_lane = reinterpret_cast<const uint8_t*>(row + kRowHeader + d.rule_width)[lane];
  } else if (sc == XMG_SCENARIO_FOUR_ROOMS) {
    nobj = 1;
    obj_lane = kGreenGoal;
  }
  // base cells of this scenario (a byte per lane: measured faster in the
  // rollout kernel than 16-byte read-only loads)
  for (int i = lane; i < HW; i += 32) ws.grid[i] = d.base_cells[i];
  if (sc == XMG_SCENARIO_EMPTY) {  // ref:scenarios.py:320-327
    __syncwarp();
    for (int i = lane; i < HW; i += 32) gdst[i] = ws.grid[i];
    res.r = 1; res.c = 1; res.d = 1;
    res.goal = 2u | ((uint32_t)kGreenGoal << 8);
    if (lane == 0) *outp = res;
    __syncwarp();
    return;
  }
  const uint64_t k0h = key.k0h, k0l = key.k0l, k1h = key.k1h, k1l = key.k1l, k2h = key.k2h, k2l = key.k2l;

  int wall_col = -1, color = 0;
  const bool two_rooms = sc == XMG_SCENARIO_DOOR_KEY || sc == XMG_SCENARIO_UNLOCK || sc == XMG_SCENARIO_UNLOCK_PICKUP;
  if (two_rooms) {  // ref:scenarios.py:341-353, 373-385
    Words4 w = {0, 0, 0, 0};
    if (lane == 0) w = philox<2>(0, 0, kDomDraw, 0, k0h, k0l);
    const uint64_t w0 = shfl64(w.w0, 0), w1 = shfl64(w.w1, 0);
    int door_row;
    if (sc == XMG_SCENARIO_DOOR_KEY) {
      wall_col = 2 + (int)(w0 % (uint64_t)(W - 4));
      door_row = 1 + (int)(w1 % (uint64_t)(H - 2));
      color = 7;  // yellow
    } else {
      wall_col = (W - 1) / 2;
      door_row = 1 + (int)(w0 % (uint64_t)(H - 2));
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
  // doors: ref:layouts.py:532-544 (segments never hold free cells)
  if (lane < nseg) {
    const int off = d.seg_off[lane], len = d.seg_off[lane + 1] - off;
    const int pos = d.fixed_doors ? len / 2 : (int)(ws.misc[2 * lane] % (uint64_t)len);
    ws.grid[d.seg_cells[off + pos]] = (uint8_t)(kClosed * 16 + cGenColors[ws.misc[2 * lane + 1] % 10]);
  }
  const uint64_t a0 = ws.misc[24], a1 = ws.misc[25];
  res.d = (int)(a1 & 3);  // a1 % 4
  if (sc == XMG_SCENARIO_XLAND || sc == XMG_SCENARIO_FOUR_ROOMS || sc == XMG_SCENARIO_EMPTY_RANDOM) {
    if (sc != XMG_SCENARIO_XLAND) res.goal = 2u | ((uint32_t)kGreenGoal << 8);  // ref:scenarios.py:330-370
    rank_place(ws, lane, F, W, 0, 0, obj_lane, nobj, nobj, a0);
  } else {  // two-room ports: shuffle all free cells, keep the left room
    rank_place(ws, lane, F, W, 1, wall_col, kKey * 16 + color, 1, 1, a0);
    if (sc == XMG_SCENARIO_DOOR_KEY) {
      res.goal = 2u | ((uint32_t)kGreenGoal << 8);
    } else if (sc == XMG_SCENARIO_UNLOCK) {  // ref:scenarios.py:393-397
      res.goal = 2u | ((uint32_t)(kOpen * 16 + color) << 8);
    } else {  // UNLOCK_PICKUP, ref:scenarios.py:400-412: reshuffle with the key placed
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
  for (int i = lane; i < HW; i += 32) gdst[i] = ws.grid[i];
  if (lane == 0) *outp = res;
  __syncwarp();
  XMG_TRB(5);
}

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
constexpr int kQueues = 128;
constexpr int kWorkHeader = 4 * kQueues;
__host__ __device__ inline int count_index(uint32_t parity, int kind, int q) {
  return (int)((parity & 1) * 2 * kQueues + kind * kQueues + q);
}
constexpr uint32_t kQPut = 1u << 31, kQReset = 1u << 30, kQEnv = (1u << 30) - 1;

// capacity of one sub-queue: every env of the step_main CTAs (128 envs each) feeding it
__host__ __device__ inline int64_t queue_cap(int64_t n) {
  const int64_t blocks = (n + kThreads - 1) / kThreads;
  return (blocks + kQueues - 1) / kQueues * kThreads;
}

// Entry slots of sub-queue (parity, kind, q): double-buffered like the counts,
// so step t + 1's step_main appends while step t's step_rare still drains.
__host__ __device__ inline int64_t queue_base(int64_t n, uint32_t parity, int kind, int q) {
  return kWorkHeader + ((int64_t)(parity & 1) * 2 * kQueues + kind * kQueues + q) * queue_cap(n);
}

// Chunk bookkeeping after the queues (chunk = the 32 envs of one step_main warp):
//   pending[nchunks]  queued envs of the chunk step_rare has not finished yet
//   dirty[nchunks]    epoch of the last step that queued envs of the chunk
// Only the chunk's own warp reads and writes its dirty word, so the tag needs
// no clearing.
__host__ __device__ inline int64_t num_chunks(int64_t n) { return (n + kThreads - 1) / kThreads * kWarps; }
__host__ __device__ inline int64_t pending_base(int64_t n) { return kWorkHeader + 4 * kQueues * queue_cap(n); }
__host__ __device__ inline int64_t dirty_base(int64_t n) { return pending_base(n) + num_chunks(n); }
__host__ __device__ inline int64_t work_words(int64_t n) { return pending_base(n) + 2 * num_chunks(n); }

__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ ulonglong2 ld_cg_u64x2(const ulonglong2* p) {  // fresh from L2, not CSE'd
  ulonglong2 v;
  asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
  return v;
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

// Per-CTA episode statistics slot (ref RolloutStats, harness.py:314-354).
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

struct MainGeo {
  int ob, stg, rb;
  int64_t total;
};

__host__ __device__ inline MainGeo make_main_geo(int V, int maxch, int R) {
  MainGeo g;
  g.ob = 2 * V * V;
  g.stg = 16 * maxch + 16;
  // per-lane rule row; after the rule pass the warp's 32 rule rows hold its
  // 32 observation records (the staging area of the bulk store)
  g.rb = max(16 * ((kRowHeader + R + 3) / 4), round16(g.ob));
  g.total = (int64_t)kThreads * (g.stg + g.rb);
  return g;
}

// abort iff *flag == epoch: xmg_validate_actions tags a rejected batch with
// the epoch of its step (atomicMax), so the flag never needs clearing.
__device__ __forceinline__ bool batch_rejected(const uint32_t* flag, uint32_t epoch) {
  return flag != nullptr && *reinterpret_cast<volatile const uint32_t*>(flag) == epoch;
}

// FULL: small grids are staged whole, issued before the state word arrives
// (one DRAM round trip per env instead of two: state word -> view window).
template <int MAXCH, bool FULL>
__global__ void __launch_bounds__(kThreads, XMG_MINB) step_main(const xmg_env_desc d, const xmg_state s,
                                                                const xmg_out o, const void* actions, int act_dtype,
                                                                const uint32_t* abort_flag, uint32_t epoch,
                                                                int64_t n) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Launched as a programmatic dependent of the previous kernel (the previous
  // step's step_rare, or this step's validation), so it runs concurrently with
  // the previous step_rare: with a validation it waits for the verdict, and
  // per 32-env chunk it waits only where the previous step queued envs (below).
  if (abort_flag != nullptr) {  // this epoch's validation verdict (published by its last CTA)
    if (lane == 0)
      for (uint32_t spins = 0; ld_acquire(abort_flag + 1) != epoch; ++spins) {
        if (spins > (1u << 25)) __trap();
        __nanosleep(64);
      }
    __syncwarp();
  }
  // the previous step_rare has read these counts (it reads them before it
  // lets this grid launch); this step appends to the other parity
  if (blockIdx.x == 0)
    for (int i = tid; i < 2 * kQueues; i += blockDim.x) s.work[count_index(epoch + 1, 0, 0) + i] = 0;
  if (batch_rejected(abort_flag, epoch)) return;

  const int H = d.height, W = d.width, HW = H * W, V = d.view_size, R = d.rule_width;
  const MainGeo geo = make_main_geo(V, MAXCH, R);
  const int64_t tile = blockIdx.x;
  const int64_t e0 = tile * kThreads;
  const int64_t chunk = tile * kWarps + warp;
  uint32_t* pending = s.work + pending_base(n) + chunk;
  uint32_t* dirty = s.work + dirty_base(n) + chunk;
  const int64_t e = e0 + tid;
  const bool valid = e < n;

  uint8_t* rb_base = smem + kThreads * geo.stg;
  uint8_t* obs_stage = rb_base + warp * 32 * geo.rb;  // aliases the warp's rule rows
  WView vw;
  vw.g = s.grids + (valid ? e : 0) * (int64_t)HW;
  vw.stage = smem + tid * geo.stg;
  vw.sbase = vw.slo = vw.shi = 0;
  uint32_t* rbuf = reinterpret_cast<uint32_t*>(rb_base + tid * geo.rb);
  if (FULL && valid) stage_issue<MAXCH>(vw, 0, HW, HW);

  // ---- load: the 16-byte state word and the action
  ulonglong2 ag = make_ulonglong2(0, 0);
  int act = 1;
  const uint32_t was_dirty = e0 + warp * 32 < n ? *dirty : 0u;  // issued together with the state loads
  if (valid) {
    ag = reinterpret_cast<const ulonglong2*>(s.agent)[e];
    act = load_action(actions, act_dtype, e);
  }
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
    if (FULL && valid) {  // the early grid copy may predate step_rare's writes
      cp_async_wait_all();
      stage_issue<MAXCH>(vw, 0, HW, HW);
    }
  }
  int r = (int)(ag.x & 0xff), c = (int)((ag.x >> 8) & 0xff), dir = (int)((ag.x >> 16) & 3);
  int pocket = (int)((ag.x >> 24) & 0xff);
  uint32_t sc = (uint32_t)(ag.x >> 32);
  const uint32_t goal_word = (uint32_t)ag.y;
  const int task = (int)(ag.y >> 32);

  uint32_t qflags = 0;
  float rew = 0.f;
  bool last = false;
  if (valid) {
    // ---- stage the post-action window (MOVE: both candidate poses) and,
    // for actions that can raise an event, the env's rule row
    const int nd = act == 1 ? ((dir + 3) & 3) : (act == 2 ? ((dir + 1) & 3) : dir);
    if (!FULL) {
      int lo, hi;
      window_span(r, c, nd, act == 0 ? 1 : 0, act == 3 ? 1 : 0, H, W, V, lo, hi);
      stage_issue<MAXCH>(vw, lo, hi, HW);
    }
    const bool rules_needed = R > 0 && (act == 0 || act == 3);
    if (rules_needed) {
      const uint32_t* src = d.task_rows + (int64_t)task * d.row_words;
      const int nq = (kRowHeader + R + 3) >> 2;
      for (int q = 0; q < nq; ++q) cp_async16(rbuf + 4 * q, src + 4 * q);
    }
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
      const int nr = R > 0 ? (int)(rbuf[1] & 0xff) : 0;
      if (nr) {
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
    if (ev == 2) {
      qflags = kQPut;  // rules, goal and reward resolved by step_rare
    } else {
      last = goal || sc >= (uint32_t)d.budget;
      if (goal) rew = goal_reward(sc, d.budget);
      o.reward[e] = rew;
      o.discount[e] = last ? 0.f : 1.f;
      o.step_type[e] = last ? 2 : 1;
      if (last) qflags = kQReset;
    }
    s.agent[2 * e] = pack_agent(r, c, dir, pocket, sc);
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
        s.work[queue_base(n, epoch, kind, k) + base + __popc(km & ((1u << lane) - 1))] = (uint32_t)e;
      }
    }
  }

  // ---- episode statistics of the trials decided here
  if (o.stats != nullptr) warp_stats(o.stats, (int)tile, rew, last ? 1.0 : 0.0, last ? (double)sc : 0.0);


  // ---- observation: assembled in smem, one TMA bulk store per warp
  // (envs queued for step_rare get theirs rewritten there)
  if (o.obs != nullptr) {
    __syncwarp();  // every lane is done with its rule row
    if (valid) {
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
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   ::"l"(gdst), "r"(saddr), "r"(bulk) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    for (uint32_t k = bulk + lane; k < bytes; k += 32) gdst[k] = obs_stage[k];
    if (lane == 0 && bulk) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

// ------------------------------------------------------- step_rare
// Observation of pose (r, c, d) on a shared-memory grid copy G, by one lane
// (lane_obs) or one view cell per lane (warp_obs), written straight to the
// env's (v, v, 2) record.
__device__ __forceinline__ uint16_t obs_cell(const uint8_t* G, int r, int c, int d, int H, int W, int V, int cell,
                                             bool see) {
  const int h = V / 2;
  const int fr = dir_dr(d), fc = dir_dc(d), rr = fc, rc = -fr;
  const int i = cell / V, j = cell - (cell / V) * V;
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

// The PUT_DOWN rule pass then the goal (ref:goals.py:347-394) of one env,
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

constexpr int kPutBatch = 8;  // PUT_DOWN envs a step_rare warp prefetches together
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
__device__ __forceinline__ void warp_reset_env(const xmg_env_desc& d, const xmg_env_desc* sd, const xmg_state& s,
                                               const xmg_out& o, uint8_t* wbase, const RareGeo& geo, int lane,
                                               int64_t e, const TrialKeys* key, int task, bool reset_mode,
                                               ResetOut* rs) {
  const int H = d.height, W = d.width, HW = H * W, V = d.view_size, ob = 2 * V * V;
  const WarpScratch ws = make_scratch(wbase, geo.hwp);
  const uint32_t g_in = d.scenario == XMG_SCENARIO_XLAND ? d.task_rows[(int64_t)task * d.row_words] : 0u;
  warp_build(sd, wbase, geo.hwp, lane, key, task, g_in, s.grids + e * (int64_t)HW, rs);
  const ResetOut ro = *rs;
  if (lane == 0) {
    reinterpret_cast<ulonglong2*>(s.rng)[e] = make_ulonglong2(ro.st_hi, ro.st_lo);
    reinterpret_cast<ulonglong2*>(s.agent)[e] = make_ulonglong2(
        pack_agent(ro.r, ro.c, ro.d, 0, 0), (uint64_t)ro.goal | ((uint64_t)(uint32_t)ro.task << 32));
    if (reset_mode) {
      o.reward[e] = 0.f;
      o.discount[e] = 1.f;
      o.step_type[e] = 0;
    }
  }
  if (o.obs != nullptr) warp_obs(ws.grid, o.obs + e * ob, lane, ro.r, ro.c, ro.d, H, W, V, d.see_through_walls != 0);
  __syncwarp();
  XMG_TRB(6);
}

// Resets of a group of up to 32 envs (one per lane, `mine`): each lane
// derives its env's trial keys, then the warp rebuilds the envs one by one.
__device__ __forceinline__ void warp_reset_group(const xmg_env_desc& d, const xmg_env_desc* sd, const xmg_state& s,
                                                 const xmg_out& o, uint8_t* wbase, const RareGeo& geo,
                                                 TrialKeys* keys, int lane, bool mine, int64_t e,
                                                 const uint64_t* reset_keys, int gw = 0) {
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
    if (in) derive_trial_keys(ek.x, ek.y, resample, keys + (lane - half));
    uint32_t m = __ballot_sync(0xffffffffu, in);
    __syncwarp();
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      const int64_t es = (int64_t)__shfl_sync(0xffffffffu, (unsigned long long)e, src);
      const int ts = __shfl_sync(0xffffffffu, task, src);
      warp_reset_env(d, sd, s, o, wbase, geo, lane, es, keys + (src - half), ts, reset_keys != nullptr,
                     reinterpret_cast<ResetOut*>(make_scratch(wbase, geo.hwp).misc + 40));
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
__global__ void __launch_bounds__(kRareWarps * 32, XMG_MINB_RARE * kWarps / kRareWarps) step_rare(const xmg_env_desc d, const xmg_state s,
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
    cnt_put = s.work[count_index(epoch, 0, q)];
    cnt_reset = s.work[count_index(epoch, 1, q)];
    if (cnt_reset > 0 && per_q < 2) {  // a single warp per sub-queue does both
      rs_w = per_q;
      jr = j;
    } else if (cnt_reset > 0) {
      if (cnt_put == 0) {
        rs_w = per_q;
      } else {
        const double wr = 4.0 * (double)cnt_reset, wp = (double)cnt_put;
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
      int off_l = 0;
      if (mine) {
        e_l = qp[it];
        const uintptr_t g0 = reinterpret_cast<uintptr_t>(s.grids + e_l * (int64_t)HW);
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
        const int res = warp_put_env(G, s.grids + e * (int64_t)HW, pc, lane, H, W, r, c, rt + kRowHeader, nr,
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
            const int slot = (int)(e / kThreads);
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
      // ---- trials the PUT_DOWN finished: keys derived one env per lane, then
      // the envs rebuilt by the whole warp
      if (lastm) {
        if ((lastm >> lane) & 1) {
          const ulonglong2 ek = reinterpret_cast<const ulonglong2*>(s.rng)[e_l];
          derive_trial_keys(ek.x, ek.y, resample, keys + lane);
        }
        __syncwarp();
        while (lastm) {
          const int src = __ffs(lastm) - 1;
          lastm &= lastm - 1;
          const int64_t es = (int64_t)__shfl_sync(0xffffffffu, (unsigned long long)e_l, src);
          const int ts = (int)(pa[src].y >> 32);
          warp_reset_env(d, sdesc, s, o, wbase, geo, lane, es, keys + src, ts, false,
                         reinterpret_cast<ResetOut*>(ws.misc + 40));
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
      const int64_t e = mine ? (int64_t)qp[i] : 0;
      warp_reset_group(d, sdesc, s, o, wbase, geo, keys, lane, mine, e, nullptr, gw);
      if (track) release_envs(s.work + pending_base(n), mine, e);
    }
  }
#ifdef XMG_TRACE
  XMG_TR(gw, 2, gtime());
#endif
}

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
  if (dyn + (int64_t)fa.sharedSizeBytes > kMaxDynSmem + 1024) return cudaErrorInvalidValue;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem - (int)fa.sharedSizeBytes);
}

// XMG_PDL=0 turns the programmatic (overlapped) launches off
bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* v = getenv("XMG_PDL");
    on = (v && !strcmp(v, "0")) ? 0 : 1;
  }
  return on == 1;
}

template <int MAXCH, bool FULL>
int launch_main(const xmg_env_desc* d, const xmg_state* s, const xmg_out* o, const void* actions, int dtype,
                const uint32_t* flag, uint32_t epoch, int64_t n, cudaStream_t st) {
  const MainGeo geo = make_main_geo(d->view_size, MAXCH, d->rule_width);
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] { attr_err = allow_smem(step_main<MAXCH, FULL>, kMaxDynSmem - 1024); });
  if (attr_err != cudaSuccess) return fail(std::string("step_main attributes: ") + cudaGetErrorString(attr_err));
  const int64_t blocks = (n + kThreads - 1) / kThreads;
  // programmatic dependent of the previous kernel on the stream (the previous
  // step's step_rare, or this step's validation)
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = (size_t)geo.total;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t err = cudaLaunchKernelEx(&cfg, step_main<MAXCH, FULL>, *d, *s, *o, actions, dtype, flag, epoch, n);
  if (err != cudaSuccess) return fail(std::string("step_main: ") + cudaGetErrorString(err));
  return check_launch("step_main");
}

// grids up to 1024 cells: the PUT_DOWN candidate lists and the radix select
// of the trial builds assume it
bool grid_fits(const xmg_env_desc* d) { return d->height * d->width <= 1024; }

int launch_rare(const xmg_env_desc* d, const xmg_state* s, const xmg_out* o, const uint64_t* keys,
                const uint32_t* flag, uint32_t epoch, int64_t n, int track, cudaStream_t st) {
  const RareGeo geo = make_rare_geo(d->height, d->width, d->rule_width);
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] { attr_err = allow_smem(step_rare, kMaxDynSmem - 1024); });
  if (attr_err != cudaSuccess) return fail(std::string("step_rare attributes: ") + cudaGetErrorString(attr_err));
  // one resident wave (warps stride over their sub-queue's entries); a
  // multiple of 32 CTAs so every sub-queue gets equal warps
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // resident CTAs per SM for this scratch size (cached: the query costs
  // microseconds of host time per launch, which small batches feel)
  static thread_local int64_t cached_smem = -1;
  static thread_local int cached_per_sm = 0;
  if (cached_smem != geo.total) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cached_per_sm, step_rare, kRareWarps * 32,
                                                      (size_t)geo.total) !=
        cudaSuccess)
      cached_per_sm = 0;
    cached_smem = geo.total;
  }
  int per_sm = cached_per_sm;
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
  step_rare<<<(unsigned)blocks, kRareWarps * 32, (size_t)geo.total, st>>>(*d, *s, *o, keys, flag, epoch, n,
                                                                                track);
  return check_launch("step_rare");
}


int validate_desc(const xmg_env_desc* d, const xmg_state* s, int64_t n) {
  if (!d) return fail("null env description");
  if (!s || !s->grids || !s->agent || !s->rng || !s->work) return fail("null state buffer");
  if (n < 1) return fail("n must be >= 1");
  if (n > (int64_t)kQEnv) return fail("n too large for one launch (< 2^30)");
  if (d->height < 1 || d->height > 255 || d->width < 1 || d->width > 255) return fail("grid size outside [1, 255]");
  if (d->view_size < 3 || !(d->view_size & 1)) return fail("view_size must be odd and >= 3");
  if (d->scenario < 0 || d->scenario > 6) return fail("unknown scenario");
  if (d->num_segments > 12) return fail("too many door segments");
  if (d->rule_width < 0 || d->rule_width > 255 || d->obj_width < 0 || d->obj_width > 255) return fail("bad widths");
  if (d->row_words < 4 || (d->row_words & 3)) return fail("row_words must be a positive multiple of 4");
  if (d->num_tasks < 1) return fail("empty task table");
  if (!d->base_cells || !d->task_rows) return fail("null base_cells / task_rows");
  if (pick_maxch(d) == 0) return fail("view window too wide for this build (v*W + v > 482)");
  if (!grid_fits(d)) return fail("grid too large for this build (H*W <= 1024)");
  if (make_main_geo(d->view_size, pick_maxch(d), d->rule_width).total > kMaxDynSmem - 1024 ||
      make_rare_geo(d->height, d->width, d->rule_width).total > kMaxDynSmem - 1024)
    return fail("grid too large for the shared-memory scratch of this build (H*W <= ~3000)");
  return 0;
}

// whole-grid staging: 16-byte chunks of a grid at any alignment
inline int full_chunks(int hw) { return (hw + 30) / 16; }

bool use_full(const xmg_env_desc* d) {
  static int mode = -1;  // XMG_STAGE=full (<= 12 chunks) | window (default: measured faster at C3)
  if (mode < 0) {
    const char* m = getenv("XMG_STAGE");
    mode = (m && !strcmp(m, "full")) ? 1 : 0;
  }
  return mode == 1 && full_chunks(d->height * d->width) <= 12;
}

int dispatch_main(const xmg_env_desc* d, const xmg_state* s, const xmg_out* o, const void* actions, int dtype,
                  const uint32_t* flag, uint32_t epoch, int64_t n, cudaStream_t st) {
  if (use_full(d)) {
    const int fc = full_chunks(d->height * d->width);
    if (fc <= 6) return launch_main<6, true>(d, s, o, actions, dtype, flag, epoch, n, st);
    if (fc <= 8) return launch_main<8, true>(d, s, o, actions, dtype, flag, epoch, n, st);
    return launch_main<12, true>(d, s, o, actions, dtype, flag, epoch, n, st);
  }
  switch (pick_maxch(d)) {
    case 6: return launch_main<6, false>(d, s, o, actions, dtype, flag, epoch, n, st);
    case 8: return launch_main<8, false>(d, s, o, actions, dtype, flag, epoch, n, st);
    case 12: return launch_main<12, false>(d, s, o, actions, dtype, flag, epoch, n, st);
    case 16: return launch_main<16, false>(d, s, o, actions, dtype, flag, epoch, n, st);
    default: return launch_main<32, false>(d, s, o, actions, dtype, flag, epoch, n, st);
  }
}

int launch_rollout(const xmg_env_desc* d, const xmg_state* s, const uint64_t* pkeys, const uint8_t* actions,
                   int64_t t0, int64_t steps, int64_t n, const xmg_out* o, cudaStream_t st) {
  const RollGeo geo = make_roll_geo(d->height, d->width, d->view_size, d->rule_width);
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] { attr_err = allow_smem(rollout_kernel, kMaxDynSmem - 1024); });
  if (attr_err != cudaSuccess) return fail(std::string("rollout_kernel attributes: ") + cudaGetErrorString(attr_err));
  if (geo.total > kMaxDynSmem - 1024) return fail("grid too large for the rollout kernel's shared-memory state");
  const int64_t chunks = (n + 31) / 32;
  const int64_t blocks = (chunks + kRollWarps - 1) / kRollWarps;
  rollout_kernel<<<(unsigned)blocks, kRollWarps * 32, (size_t)geo.total, st>>>(*d, *s, pkeys, actions, t0, steps, n,
                                                                             *o);
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

void xmg_fold_in(uint64_t hi, uint64_t lo, uint64_t data, int32_t domain, uint64_t* out2) {
  const uint64_t ctr[4] = {data, 0, (uint64_t)domain, 0};
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
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n + 4095) / 4096, sms));
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
  if (prof) cudaEventRecord(ev[0], (cudaStream_t)stream);
  if (dispatch_main(desc, state, out, actions, action_dtype, abort_flag, epoch, n, (cudaStream_t)stream)) return -1;
  if (prof) cudaEventRecord(ev[1], (cudaStream_t)stream);
  // step_main (window mode) records the tiles step_rare must release
  const int track = 1;
  const int rc = launch_rare(desc, state, out, nullptr, abort_flag, epoch, n, track, (cudaStream_t)stream);
  if (prof) cudaEventRecord(ev[2], (cudaStream_t)stream);
  return rc;
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
    if (dispatch_main(desc, state, &o, a, action_dtype, nullptr, ep, n, (cudaStream_t)stream)) return -1;
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
  const int64_t a = make_main_geo(desc->view_size, pick_maxch(desc), desc->rule_width).total;
  const int64_t b = make_rare_geo(desc->height, desc->width, desc->rule_width).total;
  return a > b ? a : b;
}

int64_t xmg_work_words(int64_t n) { return work_words(n); }

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
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
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
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
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
