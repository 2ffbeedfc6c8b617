/*
 * xmg_render_oracle.c — CPU restatement of the reference's observation images.
 *
 * TEST INFRASTRUCTURE ONLY (the checker of the device image kernel; linked by
 * tests/ through oracle/oracle.py, never by the product path).
 *
 * Restates /root/reference/pkg/src/rulegrid/render.py (cited `ref:render.py:<line>`):
 * procedural sprites (_build_sprite, :107-155) and the fixed 224x224
 * observation image (image_observation, :225-243).  The sprite masks are
 * evaluated in IEEE double with one rounding per operation, in NumPy's order
 * (build with -ffp-contract=off), so every comparison lands on the same side
 * as in the reference.  Pinned by tests/golden/render_golden.json (digests of
 * the reference's own sprites and images, tests/golden/make_render_golden.py).
 */
#include <stdint.h>
#include <string.h>

enum { T_EOM = 0, T_UNSEEN, T_EMPTY, T_FLOOR, T_WALL, T_BALL, T_SQUARE, T_PYRAMID, T_GOAL, T_KEY,
       T_DOOR_LOCKED, T_DOOR_CLOSED, T_DOOR_OPEN, T_HEX, T_STAR };

#define IMAGE_SIDE 224 /* ref:render.py:21 */

/* ref:render.py:48-63 (_COLOR_RGB), :65-67 (_BG, _GRID_LINE, _UNSEEN_SHADE) */
static const uint8_t COLOR_RGB[14][3] = {
    {0, 0, 0},       {12, 12, 12},   {0, 0, 0},      {220, 50, 50},  {60, 180, 75},
    {65, 105, 225},  {145, 70, 200}, {235, 200, 50}, {150, 150, 150}, {25, 25, 25},
    {240, 140, 40},  {245, 245, 245}, {150, 100, 60}, {240, 130, 180}};
static const uint8_t BG[3] = {30, 30, 30};
static const uint8_t GRID_LINE[3] = {45, 45, 45};

static double fabs_(double x) { return x < 0 ? -x : x; }

static void put(uint8_t* px3, const uint8_t rgb[3]) { px3[0] = rgb[0]; px3[1] = rgb[1]; px3[2] = rgb[2]; }

/* One pixel (y, x) of sprite (tile, color, px): ref:render.py:107-155, with
 * the masks of _shape_masks (:96-100): dy = (y - cy) / px, cy = (px - 1) / 2. */
static void sprite_pixel(int tile, int color, int px, int y, int x, uint8_t out[3]) {
  const uint8_t* rgb = COLOR_RGB[color];
  const double cy = (px - 1) / 2.0;
  const double dy = ((double)y - cy) / (double)px, dx = ((double)x - cy) / (double)px;
  uint8_t half[3], tq[3], black[3] = {0, 0, 0};
  for (int k = 0; k < 3; ++k) { half[k] = rgb[k] / 2; tq[k] = (uint8_t)(rgb[k] * 3 / 4); }
  put(out, BG);
  switch (tile) {
    case T_EOM: case T_EMPTY: put(out, black); break;
    case T_UNSEEN: put(out, COLOR_RGB[1]); break;
    case T_FLOOR:
      if (y == px - 1 || x == px - 1) {  /* grid line tinted with the floor color */
        uint8_t line[3];
        for (int k = 0; k < 3; ++k) line[k] = (uint8_t)((GRID_LINE[k] + rgb[k]) / 2);
        put(out, line);
      }
      break;
    case T_WALL: put(out, rgb); break;
    case T_BALL: if (dy * dy + dx * dx <= 0.35 * 0.35) put(out, rgb); break;
    case T_SQUARE: if (fabs_(dy) <= 0.30 && fabs_(dx) <= 0.30) put(out, rgb); break;
    case T_PYRAMID: if (dy >= -0.35 && dy <= 0.35 && fabs_(dx) <= (dy + 0.35) / 2) put(out, rgb); break;
    case T_GOAL: {
      const int e = px / 8 + 1;
      const int edge = (y < e) || (y >= px - px / 8 - 1) || (x < e) || (x >= px - px / 8 - 1);
      put(out, edge ? rgb : half);
      break;
    }
    case T_KEY: {
      if (fabs_(dx) <= 0.13 && dy >= -0.15 && dy <= 0.38) put(out, rgb);
      const double a = dy + 0.22;
      const double ring = dx * dx + a * a;
      if (ring <= 0.18 * 0.18 && ring >= 0.08 * 0.08) put(out, rgb);
      if (fabs_(dy - 0.30) <= 0.05 && dx >= 0.0 && dx <= 0.2) put(out, rgb);
      break;
    }
    case T_DOOR_LOCKED: case T_DOOR_CLOSED: case T_DOOR_OPEN: {
      const int frame = fabs_(dy) >= 0.36 || fabs_(dx) >= 0.36;
      if (frame) put(out, rgb);
      if (tile == T_DOOR_LOCKED) {
        if (!frame) put(out, half);
        if (dy * dy + dx * dx <= 0.07 * 0.07) put(out, black);
      } else if (tile == T_DOOR_CLOSED) {
        if (!frame) put(out, tq);
        const double b = dx - 0.22;
        if (b * b + dy * dy <= 0.06 * 0.06) put(out, black);
      }
      break;
    }
    case T_HEX: if (fabs_(dy) <= 0.32 && fabs_(dx) + 0.5 * fabs_(dy) <= 0.38) put(out, rgb); break;
    case T_STAR: {
      const int spokes = fabs_(dx) <= 0.09 || fabs_(dy) <= 0.09;
      if (spokes && fabs_(dx) + fabs_(dy) <= 0.42) put(out, rgb);
      if (fabs_(dx) + fabs_(dy) <= 0.16) put(out, rgb);
      break;
    }
    default: break;
  }
}

/* ref:render.py:158-169 (sprite): (px, px, 3) u8; returns -1 for px < 4 or a
 * code outside the enums (the reference raises). */
int32_t xmgo_sprite(int32_t tile, int32_t color, int32_t px, uint8_t* out) {
  if (px < 4 || tile < 0 || tile > 14 || color < 0 || color > 13) return -1;
  for (int y = 0; y < px; ++y)
    for (int x = 0; x < px; ++x) sprite_pixel(tile, color, px, y, x, out + 3 * (y * px + x));
  return 0;
}

/* ref:render.py:225-243 (image_observation) for n observations (v, v, 2):
 * px = 224 // v, margin (224 - v*px) // 2 in the UNSEEN shade, cell (r, c)
 * drawn with sprite(obs[r][c]). */
int32_t xmgo_image_observations(const uint8_t* obs, int64_t n, int32_t v, uint8_t* out) {
  const int px = IMAGE_SIDE / v;
  if (v < 1 || px < 4) return -1;
  const int off = (IMAGE_SIDE - v * px) / 2;
  static uint8_t cache[15 * 14][74 * 74 * 3];
  static int cache_px = -1;
  if (px > 74) return -1;
  if (cache_px != px) {
    for (int t = 0; t < 15; ++t)
      for (int c = 0; c < 14; ++c) xmgo_sprite(t, c, px, cache[t * 14 + c]);
    cache_px = px;
  }
  for (int64_t e = 0; e < n; ++e) {
    uint8_t* img = out + e * (int64_t)IMAGE_SIDE * IMAGE_SIDE * 3;
    for (int i = 0; i < IMAGE_SIDE * IMAGE_SIDE; ++i) put(img + 3 * i, COLOR_RGB[1]);
    const uint8_t* o = obs + e * (int64_t)v * v * 2;
    for (int r = 0; r < v; ++r)
      for (int c = 0; c < v; ++c) {
        const int t = o[2 * (r * v + c)], col = o[2 * (r * v + c) + 1];
        if (t > 14 || col > 13) return -1;
        const uint8_t* sp = cache[t * 14 + col];
        for (int y = 0; y < px; ++y)
          memcpy(img + 3 * ((off + r * px + y) * IMAGE_SIDE + off + c * px), sp + 3 * y * px, 3 * (size_t)px);
      }
  }
  return 0;
}
