// xmg_render.cuh — 224x224 RGB observation images on the device (included by
// xmg_step.cu inside its anonymous namespace).
//
// ref:render.py (cited below): procedural sprites (_build_sprite :107-155),
// cached per (tile, color, px) (:158-169), and image_observation (:225-243):
// px = 224 // v, the v*px square centred with an UNSEEN-shade margin, cell
// (r, c) drawn with sprite(obs[r][c]).
//
// Two kernels:
//  * sprite_kernel builds the whole atlas [15 tiles][14 colors][px][px][3]
//    for one px, one thread per pixel; the masks are evaluated in IEEE double
//    with one rounding per operation in NumPy's order (explicit _rn
//    intrinsics: no FMA contraction), so every pixel equals the reference's;
//  * image_kernel writes images: a CTA of 168 threads renders one image at a
//    time, thread w owning 4-byte word w of every row; a word is one or two
//    unaligned 4-byte reads of the atlas (L2-resident, 1.2 MB at px = 44)
//    merged with byte_perm.  HBM-write bound: 150528 bytes out per image,
//    v*v*2 in.

constexpr int kImageSide = 224;
constexpr int kImageRow = 3 * kImageSide;          // 672 bytes
constexpr int kImageBytes = kImageSide * kImageRow;  // 150528

// ref:render.py:48-67: _COLOR_RGB, _BG, _GRID_LINE
__constant__ uint8_t cColorRGB[14][3] = {
    {0, 0, 0},      {12, 12, 12},  {0, 0, 0},       {220, 50, 50},  {60, 180, 75},
    {65, 105, 225}, {145, 70, 200}, {235, 200, 50}, {150, 150, 150}, {25, 25, 25},
    {240, 140, 40}, {245, 245, 245}, {150, 100, 60}, {240, 130, 180}};

__device__ __forceinline__ double dsq(double a) { return __dmul_rn(a, a); }

// One pixel of sprite (tile, color, px), packed 0x00BBGGRR.
__device__ uint32_t sprite_pixel(int tile, int color, int px, int y, int x) {
  const uint32_t rgb = cColorRGB[color][0] | (cColorRGB[color][1] << 8) | (cColorRGB[color][2] << 16);
  auto pack = [](int r, int g, int b) { return (uint32_t)r | ((uint32_t)g << 8) | ((uint32_t)b << 16); };
  const int R = cColorRGB[color][0], G = cColorRGB[color][1], B = cColorRGB[color][2];
  const uint32_t half = pack(R / 2, G / 2, B / 2), tq = pack(R * 3 / 4, G * 3 / 4, B * 3 / 4);
  const uint32_t bg = pack(30, 30, 30), black = 0;
  // _shape_masks (:96-100): dy = (y - cy) / px, cy = cx = (px - 1) / 2.0
  const double cy = __ddiv_rn((double)(px - 1), 2.0);
  const double dy = __ddiv_rn(__dsub_rn((double)y, cy), (double)px);
  const double dx = __ddiv_rn(__dsub_rn((double)x, cy), (double)px);
  const double ady = fabs(dy), adx = fabs(dx);
  const double r2 = __dadd_rn(dsq(dy), dsq(dx));
  uint32_t out = bg;
  switch (tile) {
    case 0: case 2: out = black; break;                       // END_OF_MAP, EMPTY
    case 1: out = pack(12, 12, 12); break;                    // UNSEEN
    case 3:                                                   // FLOOR: tinted grid line
      if (y == px - 1 || x == px - 1) out = pack((45 + R) / 2, (45 + G) / 2, (45 + B) / 2);
      break;
    case 4: out = rgb; break;                                 // WALL
    case 5: if (r2 <= __dmul_rn(0.35, 0.35)) out = rgb; break;  // BALL
    case 6: if (ady <= 0.30 && adx <= 0.30) out = rgb; break;   // SQUARE
    case 7:                                                     // PYRAMID
      if (dy >= -0.35 && dy <= 0.35 && adx <= __ddiv_rn(__dadd_rn(dy, 0.35), 2.0)) out = rgb;
      break;
    case 8: {                                                   // GOAL
      const int e = px / 8 + 1, f = px - px / 8 - 1;
      out = (y < e || y >= f || x < e || x >= f) ? rgb : half;
      break;
    }
    case 9: {                                                   // KEY
      if (adx <= 0.13 && dy >= -0.15 && dy <= 0.38) out = rgb;
      const double ring = __dadd_rn(dsq(dx), dsq(__dadd_rn(dy, 0.22)));
      if (ring <= __dmul_rn(0.18, 0.18) && ring >= __dmul_rn(0.08, 0.08)) out = rgb;
      if (fabs(__dsub_rn(dy, 0.30)) <= 0.05 && dx >= 0.0 && dx <= 0.2) out = rgb;
      break;
    }
    case 10: case 11: case 12: {                                // doors
      const bool frame = ady >= 0.36 || adx >= 0.36;
      if (frame) out = rgb;
      if (tile == 10) {
        if (!frame) out = half;
        if (r2 <= __dmul_rn(0.07, 0.07)) out = black;
      } else if (tile == 11) {
        if (!frame) out = tq;
        if (__dadd_rn(dsq(__dsub_rn(dx, 0.22)), dsq(dy)) <= __dmul_rn(0.06, 0.06)) out = black;
      }
      break;
    }
    case 13:                                                    // HEX
      if (ady <= 0.32 && __dadd_rn(adx, __dmul_rn(0.5, ady)) <= 0.38) out = rgb;
      break;
    case 14: {                                                  // STAR
      const bool spokes = adx <= 0.09 || ady <= 0.09;
      const double l1 = __dadd_rn(adx, ady);
      if (spokes && l1 <= 0.42) out = rgb;
      if (l1 <= 0.16) out = rgb;
      break;
    }
    default: break;
  }
  return out;
}

__global__ void sprite_kernel(int px, uint8_t* atlas) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)px * px;
  if (i >= 210 * per) return;
  const int s = (int)(i / per), p = (int)(i - s * per);
  const uint32_t v = sprite_pixel(s / 14, s % 14, px, p / px, p % px);
  uint8_t* o = atlas + 3 * i;
  o[0] = (uint8_t)v;
  o[1] = (uint8_t)(v >> 8);
  o[2] = (uint8_t)(v >> 16);
}

// Unaligned 32-bit read from the (padded) atlas: two aligned words and a
// funnel shift.
__device__ __forceinline__ uint32_t ldu32(const uint8_t* p) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uint32_t* q = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
  return __funnelshift_r(__ldg(q), __ldg(q + 1), (uint32_t)(a & 3) * 8u);
}

constexpr uint32_t kShade = 0x0C0C0C0Cu;  // UNSEEN shade (12, 12, 12) bytes
constexpr int kMarginCol = 255;

// Images of n observations (v, v, 2).  One CTA per image at a time
// (grid-stride over envs); thread w owns 4-byte word w of every image row
// (168 words, 672 bytes: a row is one coalesced 672-byte store per CTA).  A
// word shows at most two cell columns (a sprite row is 3*px >= 12 bytes): the
// thread's column pair, byte offsets and byte_perm selector are fixed for
// the whole image, so walking down the rows is a pointer increment of one
// sprite row (3*px bytes) per row and two unaligned 4-byte atlas reads
// (L1/L2 resident) per word.
constexpr int kImageWords = kImageRow / 4;  // 168

__global__ void __launch_bounds__(kImageWords) image_kernel(const uint8_t* __restrict__ obs, int64_t n, int v, int px,
                                                           const uint8_t* __restrict__ atlas,
                                                           uint8_t* __restrict__ out) {
  __shared__ uint32_t base[56 * 56];  // atlas offset of cell (r, c)'s sprite (v <= 224 / 4)
  const int w = threadIdx.x;
  const int off = (kImageSide - v * px) / 2, span = v * px, srow = 3 * px;
  // this thread's word: first / last byte's cell column (or the margin), the
  // word's byte offset inside each column's sprite row, the merge selector
  int col[2], rel[2];
  for (int k = 0; k < 2; ++k) {
    const int x = (4 * w + 3 * k) / 3 - off;
    col[k] = (x < 0 || x >= span) ? kMarginCol : x / px;
    rel[k] = col[k] == kMarginCol ? 0 : 4 * w - 3 * (off + col[k] * px);
  }
  uint32_t sel = 0;
  for (int j = 0; j < 4; ++j) {  // byte j from the first column unless it lies in the second's span
    const int x = (4 * w + j) / 3 - off;
    const int cj = (x < 0 || x >= span) ? kMarginCol : x / px;
    sel |= (uint32_t)(cj == col[0] ? j : 4 + j) << (4 * j);
  }
  const bool ma = col[0] == kMarginCol, mb = col[1] == kMarginCol, two = col[1] != col[0];
  const uint32_t spr = (uint32_t)(srow * px);
  for (int64_t e = blockIdx.x; e < n; e += gridDim.x) {
    __syncthreads();  // previous image's bases consumed
    for (int k = w; k < v * v; k += blockDim.x) {
      const int t = obs[(e * v * v + k) * 2], c = obs[(e * v * v + k) * 2 + 1];
      base[k] = (t <= 14 && c <= 13) ? (uint32_t)(t * 14 + c) * spr : 0u;  // invalid codes: END_OF_MAP
    }
    __syncthreads();
    uint32_t* o = reinterpret_cast<uint32_t*>(out + e * (int64_t)kImageBytes) + w;
    for (int Y = 0; Y < off; ++Y) o[Y * kImageWords] = kShade;
    for (int Y = off + span; Y < kImageSide; ++Y) o[Y * kImageWords] = kShade;
    o += off * kImageWords;
    for (int i = 0; i < v; ++i) {
      // rel may be negative (a word starting before its column): signed offsets
      const uint8_t* pa = atlas + (ma ? 0 : (int64_t)base[i * v + col[0]] + rel[0]);
      const uint8_t* pb = atlas + (mb ? 0 : (int64_t)base[i * v + col[1]] + rel[1]);
#pragma unroll 4
      for (int sy = 0; sy < px; ++sy) {
        const uint32_t a = ma ? kShade : ldu32(pa);
        const uint32_t b = two ? (mb ? kShade : ldu32(pb)) : a;
        *o = __byte_perm(a, b, sel);
        o += kImageWords;
        pa += srow;
        pb += srow;
      }
    }
  }
}

// ---------------------------------------------------------------- aligned path
// For views with px >= 6 (v <= 37) the image is written in 16-byte chunks
// straight from a phase-shifted copy of the atlas: column c's sprite rows
// start at image-row byte D_c = 3 * (off + c * px); their phase D_c mod 16 is
// one of at most 16 values, and the "aligned atlas" holds every sprite row
// once per phase in use, shifted right by that phase inside a row pitch of
// P = round16(3 * px + 15) bytes.  A 16-byte output chunk then shows at most
// two columns (3 * px >= 18 > 16), each one aligned 16-byte load, merged with
// byte_perm; one coalesced 16-byte store.
struct ImgGeo {
  int px, off, span, pitch, nphase;
  int phase_of[37];  // column -> phase index (first-appearance order of D_c mod 16)
  int phase_val[16];
};

__host__ __device__ inline ImgGeo make_img_geo(int v) {
  ImgGeo g;
  g.px = kImageSide / v;
  g.off = (kImageSide - v * g.px) / 2;
  g.span = v * g.px;
  g.pitch = round16(3 * g.px + 15);
  g.nphase = 0;
  for (int c = 0; c < v && c < 37; ++c) {
    const int ph = (3 * (g.off + c * g.px)) & 15;
    int k = 0;
    while (k < g.nphase && g.phase_val[k] != ph) ++k;
    if (k == g.nphase) g.phase_val[g.nphase++] = ph;
    g.phase_of[c] = k;
  }
  return g;
}

inline int64_t aligned_atlas_bytes(int v) {
  const ImgGeo g = make_img_geo(v);
  return (int64_t)g.nphase * 210 * g.px * g.pitch;
}

// aligned[p][s][sy][pitch] = sprite s row sy shifted right by phase_val[p]
__global__ void aligned_atlas_kernel(int v, const uint8_t* __restrict__ atlas, uint8_t* __restrict__ out) {
  const ImgGeo g = make_img_geo(v);
  const int64_t per_row = g.pitch, rows = (int64_t)g.nphase * 210 * g.px;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * per_row) return;
  const int64_t row = i / per_row;
  const int b = (int)(i - row * per_row);
  const int p = (int)(row / (210 * g.px));
  const int64_t sr = row - (int64_t)p * 210 * g.px;  // sprite * px + sy
  const int src = b - g.phase_val[p];
  out[i] = (src >= 0 && src < 3 * g.px) ? atlas[sr * 3 * g.px + src] : 0;
}

constexpr int kImgChunks = kImageRow / 16;   // 42 chunks of 16 bytes per row
constexpr int kImgRowsPar = 4;               // rows in flight per CTA
constexpr int kImgThreads = kImgChunks * kImgRowsPar;  // 168
constexpr int kMarginColA = 255;

#ifndef XMG_IMG_MINB
#define XMG_IMG_MINB 1
#endif
#ifndef XMG_IMG_UNROLL
#define XMG_IMG_UNROLL 4
#endif
__global__ void __launch_bounds__(kImgThreads, XMG_IMG_MINB) image_kernel_aligned(const uint8_t* __restrict__ obs, int64_t n,
                                                                    int v, const uint8_t* __restrict__ aligned,
                                                                    uint8_t* __restrict__ out) {
  __shared__ uint16_t spr[37 * 37];      // sprite index (tile * 14 + color) of cell (r, c)
  __shared__ uint16_t rowinfo[kImageSide];  // image row -> cell row << 8 | sprite row, 0xFFFF in the margin
  const ImgGeo g = make_img_geo(v);
  const int t = threadIdx.x, q = t % kImgChunks, rp = t / kImgChunks;
  for (int Y = t; Y < kImageSide; Y += blockDim.x) {
    const int yy = Y - g.off;
    rowinfo[Y] = (yy < 0 || yy >= g.span) ? (uint16_t)0xFFFF : (uint16_t)(((yy / g.px) << 8) | (yy % g.px));
  }
  // this thread's chunk: its first / last byte's column (or the margin)
  auto col_of = [&](int b) {
    const int x = b / 3 - g.off;
    return (x < 0 || x >= g.span) ? kMarginColA : x / g.px;
  };
  const int ca = col_of(16 * q), cb = col_of(16 * q + 15);
  const bool two = cb != ca;
  // first byte of cb inside the chunk
  const int tb = !two ? 16 : (cb == kMarginColA ? 3 * (g.off + g.span) : 3 * (g.off + cb * g.px)) - 16 * q;
  // per-word merge selectors: the first k = tb - 4w bytes of word w from A,
  // the rest from B (0x3210 = all A, 0x7654 = all B)
  uint32_t selw[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const int k = min(max(tb - 4 * w, 0), 4);
    uint32_t sel = 0;
    for (int j = 0; j < 4; ++j) sel |= (uint32_t)(j < k ? j : 4 + j) << (4 * j);
    selw[w] = sel;
  }
  // 32-bit atlas offsets: chunk offset inside the column's aligned row plus
  // its phase block; a sprite adds spr * sstride, a sprite row sy * pitch
  const uint32_t sstride = (uint32_t)(g.px * g.pitch);
  uint32_t baseA = 0, baseB = 0;
  if (ca != kMarginColA) {
    const int D = 3 * (g.off + ca * g.px);
    baseA = (uint32_t)(g.phase_of[ca] * 210) * sstride + (uint32_t)(16 * q - (D - g.phase_val[g.phase_of[ca]]));
  }
  if (two && cb != kMarginColA) {
    const int D = 3 * (g.off + cb * g.px);
    baseB = (uint32_t)(g.phase_of[cb] * 210) * sstride + (uint32_t)(16 * q - (D - g.phase_val[g.phase_of[cb]]));
  }
  const bool loadA = ca != kMarginColA, loadB = two && cb != kMarginColA;
  const uint32_t pitch = (uint32_t)g.pitch;
  const uint4 shade = make_uint4(kShade, kShade, kShade, kShade);
  for (int64_t e = blockIdx.x; e < n; e += gridDim.x) {
    __syncthreads();  // previous image's sprite ids consumed
    for (int k = t; k < v * v; k += blockDim.x) {
      const int tt = obs[(e * v * v + k) * 2], cc = obs[(e * v * v + k) * 2 + 1];
      spr[k] = (tt <= 14 && cc <= 13) ? (uint16_t)(tt * 14 + cc) : 0;  // invalid codes: END_OF_MAP
    }
    __syncthreads();
    uint8_t* img = out + e * (int64_t)kImageBytes + 16 * q;
    // kU rows per iteration: their loads are independent and go out together
    constexpr int kU = XMG_IMG_UNROLL;
    for (int Y0 = rp; Y0 < kImageSide; Y0 += kU * kImgRowsPar) {
      uint4 A[kU], B[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int Y = Y0 + u * kImgRowsPar;
        A[u] = B[u] = shade;
        const uint32_t info = Y < kImageSide ? rowinfo[Y] : 0xFFFFu;
        if (info != 0xFFFFu) {
          const int i = (int)(info >> 8);
          const uint32_t rowoff = (info & 0xFFu) * pitch;
          if (loadA) A[u] = __ldg(reinterpret_cast<const uint4*>(aligned + baseA + spr[i * v + ca] * sstride + rowoff));
          if (loadB) B[u] = __ldg(reinterpret_cast<const uint4*>(aligned + baseB + spr[i * v + cb] * sstride + rowoff));
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int Y = Y0 + u * kImgRowsPar;
        if (Y >= kImageSide) break;
        const uint4 a = A[u], b = B[u];  // B == shade when the chunk shows one column (selectors: all A)
        *reinterpret_cast<uint4*>(img + (int64_t)Y * kImageRow) =
            make_uint4(__byte_perm(a.x, b.x, selw[0]), __byte_perm(a.y, b.y, selw[1]),
                       __byte_perm(a.z, b.z, selw[2]), __byte_perm(a.w, b.w, selw[3]));
      }
    }
  }
}
