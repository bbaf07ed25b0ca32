/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, single-threaded CPU
 * oracle for Barnes, "Parallel Non-divergent Flow Accumulation for Trillion
 * Cell DEMs" (arXiv 1608.04431).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * path (paper_1608_04431_b200/csrc); neither includes the other.
 *
 * Citations: "P:Lnn" = /root/reference/PAPER.md line nn (section /
 * algorithm / equation named beside it); "S:Lnn" = SPEC.md line nn;
 * "Dn" = reading n in DESIGN.md ("Readings of the paper").
 *
 * Direction codes (D1): 0 NoFlow, 1 N(0,-1), 2 NE(+1,-1),
 * 3 E(+1,0), 4 SE(+1,+1), 5 S(0,+1), 6 SW(-1,+1), 7 W(-1,0), 8 NW(-1,-1),
 * 255 NoData; (dx, dy) with y growing downward (row index).
 *
 * Status codes: 0 ok, 1 bad argument, 2 illegal direction byte,
 * 3 cycle (some data cell never retires), 5 out of memory.
 *
 * Every function below is pinned by tests in tests/test_oracle_*.py
 * (see DESIGN.md "Pins"); none is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_NODATA 255
#define OR_NOFLOW 0
#define OR_FLOW_EXTERNAL 0xFFFFFFFEu
#define OR_FLOW_TERMINATES 0xFFFFFFFFu
#define OR_LINK_CYCLE 0xFFFFFFFDu

/* direction offsets, code k at index k (index 0 unused) -- S:L33 */
static const int ODX[9] = {0, 0, 1, 1, 1, 0, -1, -1, -1};
static const int ODY[9] = {0, -1, -1, 0, 1, 1, 1, 0, -1};

int or_dir_offset(int code, int* dx, int* dy) {
  if (code < 1 || code > 8) return 1;
  *dx = ODX[code];
  *dy = ODY[code];
  return 0;
}

/* ======================================================================
 * O-D8: steepest-descent D8 ("D8 ... apportion a cell's flow to a
 * single one of its neighbours"; the stencil rule is BASELINE.json
 * north_star: "ties broken by lowest neighbour index, diagonal drop divided
 * by sqrt2"; readings D2-D6 of DESIGN.md).
 * ==================================================================== */
static int o_is_nodata(float v, float nodata) { return isnan(v) || isinf(v) || v == nodata; }

void or_d8(const float* z, int64_t H, int64_t W, float nodata, uint8_t* dirs) {
  for (int64_t y = 0; y < H; ++y) {
    for (int64_t x = 0; x < W; ++x) {
      const float zc = z[y * W + x];
      /* step 1: NoData cell */
      if (o_is_nodata(zc, nodata)) {
        dirs[y * W + x] = OR_NODATA;
        continue;
      }
      /* step 2: classify neighbours, drops d_k = fl32(z - z_k) (D5) */
      int has_out = 0, first_out = 0;
      float a = 0.0f, b = 0.0f; /* best cardinal / diagonal drop */
      int kc = 0, kd = 0;
      for (int k = 1; k <= 8; ++k) {
        int64_t nx = x + ODX[k], ny = y + ODY[k];
        int outside = nx < 0 || ny < 0 || nx >= W || ny >= H;
        if (outside || o_is_nodata(z[ny * W + nx], nodata)) {
          if (!has_out) {
            has_out = 1;
            first_out = k;
          }
          continue;
        }
        float d = zc - z[ny * W + nx];
        if (!(d > 0.0f)) continue; /* strictly downhill only */
        if (k % 2 == 1) {          /* step 3: cardinal, first k wins ties */
          if (kc == 0 || d > a) {
            a = d;
            kc = k;
          }
        } else { /* step 4: diagonal */
          if (kd == 0 || d > b) {
            b = d;
            kd = k;
          }
        }
      }
      uint8_t code;
      if (kc && kd) {
        /* step 5: cardinal iff a > b/sqrt(2)  <=>  2a^2 > b^2, exact in
         * double (24-bit significands square into <= 48 bits) (D4) */
        double da = (double)a, db = (double)b;
        code = (uint8_t)((2.0 * da * da > db * db) ? kc : kd);
      } else if (kc) {
        code = (uint8_t)kc;
      } else if (kd) {
        code = (uint8_t)kd;
      } else {
        /* step 6: outlet fallback (D3) or NoFlow (D6) */
        code = (uint8_t)(has_out ? first_out : OR_NOFLOW);
      }
      dirs[y * W + x] = code;
    }
  }
}

/* index of the first illegal direction byte, or -1 (D1) */
int64_t or_validate(const uint8_t* dirs, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (dirs[i] > 8 && dirs[i] != OR_NODATA) return i;
  return -1;
}

/* target of cell (x,y) inside the region [y0,y0+h) x [x0,x0+w) of an H x W
 * raster: the neighbour named by F if F in 1..8, the neighbour lies in the
 * region and is not NoData; otherwise -1 (Alg. 1; D8; D23).   */
static int64_t o_target(const uint8_t* dirs, int64_t W, int64_t x, int64_t y, int64_t y0,
                        int64_t x0, int64_t h, int64_t w) {
  uint8_t f = dirs[y * W + x];
  if (f < 1 || f > 8) return -1;
  int64_t nx = x + ODX[f], ny = y + ODY[f];
  if (nx < x0 || ny < y0 || nx >= x0 + w || ny >= y0 + h) return -1;
  if (dirs[ny * W + nx] == OR_NODATA) return -1;
  return ny * W + nx;
}

/* ======================================================================
 * O-ACC: Eq. 1 (equ:flow_acc) with alpha in {0,1}:
 *   A(p) = w(p) + sum_{n : target(n) = p} A(n)
 * on a region treated as a whole raster ("authoritative
 * answer"), computed by Kahn's algorithm (Alg. 1) with an
 * immediate depth-first schedule: scan cells in row-major order; from each
 * unretired data cell with D = 0 follow the chain, adding A downstream and
 * continuing only while the target's dependency count reaches 0.
 * NoData cells get the marker (D9).  NoFlow cells keep inflow + own w (D7).
 * Generic over the accumulator type via a macro (u64 for integer weights,
 * double for float weights, int64 fixed point for the exact pin P11).
 * ==================================================================== */
#define OR_ACC_BODY(T, WEXPR, NDMARK)                                                    \
  const int64_t N = h * w;                                                              \
  if (h <= 0 || w <= 0) return 1;                                                       \
  for (int64_t yy = y0; yy < y0 + h; ++yy)                                              \
    for (int64_t xx = x0; xx < x0 + w; ++xx) {                                          \
      uint8_t f = dirs[yy * W + xx];                                                    \
      if (f > 8 && f != OR_NODATA) return 2;                                            \
    }                                                                                   \
  uint8_t* D = (uint8_t*)calloc((size_t)N, 1);                                          \
  if (!D) return 5;                                                                     \
  /* dependency counts: donors inside the region (Alg. 1 first loop) */                \
  int64_t ndata = 0;                                                                    \
  for (int64_t yy = y0; yy < y0 + h; ++yy)                                              \
    for (int64_t xx = x0; xx < x0 + w; ++xx) {                                          \
      int64_t i = yy * W + xx;                                                          \
      if (dirs[i] == OR_NODATA) continue;                                               \
      ++ndata;                                                                          \
      int64_t t = o_target(dirs, W, xx, yy, y0, x0, h, w);                              \
      if (t >= 0) D[((t / W) - y0) * w + (t % W) - x0]++;                              \
    }                                                                                   \
  /* A = w */                                                                           \
  for (int64_t yy = y0; yy < y0 + h; ++yy)                                              \
    for (int64_t xx = x0; xx < x0 + w; ++xx) {                                          \
      int64_t i = yy * W + xx;                                                          \
      A[i] = dirs[i] == OR_NODATA ? (NDMARK) : (WEXPR);                                 \
    }                                                                                   \
  /* Kahn with chain following; D = 255 marks a retired cell */                        \
  int64_t retired = 0;                                                                  \
  for (int64_t yy = y0; yy < y0 + h; ++yy)                                              \
    for (int64_t xx = x0; xx < x0 + w; ++xx) {                                          \
      int64_t li = (yy - y0) * w + (xx - x0);                                           \
      if (dirs[yy * W + xx] == OR_NODATA || D[li] != 0) continue;                       \
      int64_t cx = xx, cy = yy;                                                         \
      for (;;) {                                                                        \
        int64_t cl = (cy - y0) * w + (cx - x0);                                         \
        D[cl] = 255;                                                                    \
        ++retired;                                                                      \
        int64_t t = o_target(dirs, W, cx, cy, y0, x0, h, w);                            \
        if (t < 0) break;                                                               \
        A[t] += A[cy * W + cx];                                                         \
        int64_t tl = ((t / W) - y0) * w + (t % W) - x0;                                 \
        if (--D[tl] > 0) break;                                                         \
        cx = t % W;                                                                     \
        cy = t / W;                                                                     \
      }                                                                                 \
    }                                                                                   \
  free(D);                                                                              \
  return retired == ndata ? 0 : 3;

int or_acc_region_u64(const uint8_t* dirs, int64_t H, int64_t W, int64_t y0, int64_t x0,
                      int64_t h, int64_t w, const uint32_t* wt, uint64_t* A) {
  (void)H;
  OR_ACC_BODY(uint64_t, (wt ? (uint64_t)wt[i] : (uint64_t)1), UINT64_MAX)
}

int or_acc_region_f64(const uint8_t* dirs, int64_t H, int64_t W, int64_t y0, int64_t x0,
                      int64_t h, int64_t w, const float* wt, double* A) {
  (void)H;
  OR_ACC_BODY(double, (wt ? (double)wt[i] : 1.0), NAN)
}

/* exact fixed point: A in units of 2^-shift (weights must lie on that grid) */
int or_acc_region_fix(const uint8_t* dirs, int64_t H, int64_t W, int64_t y0, int64_t x0,
                      int64_t h, int64_t w, const float* wt, int shift, int64_t* A) {
  (void)H;
  const double scale = ldexp(1.0, shift);
  for (int64_t yy = y0; yy < y0 + h; ++yy)
    for (int64_t xx = x0; xx < x0 + w; ++xx) {
      double v = (double)wt[yy * W + xx] * scale;
      if (dirs[yy * W + xx] != OR_NODATA && v != floor(v)) return 1;
    }
  OR_ACC_BODY(int64_t, (int64_t)((double)wt[i] * scale), INT64_MIN)
}

/* ======================================================================
 * O-ACC with absorption: Eq. 1 with a per-cell
 * fraction alpha(n) in [0,1] of A(n) passed on to its single (non-divergent)
 * target, "flow may be absorbed during its downhill movement ... so alpha is
 * constrained such that sum_p alpha(n,p) <= 1", "most forms of
 * absorption represent a simple extension":
 *   A(p) = w(p) + sum_{n : target(n) = p} alpha(n) A(n)
 * Same Kahn schedule as O-ACC; only the push is scaled.  Returns 1 if an
 * alpha of a data cell is not a finite value in [0,1].
 * ==================================================================== */
int or_acc_alpha_f64(const uint8_t* dirs, int64_t H, int64_t W, const float* wt, const float* alpha,
                     double* A) {
  const int64_t y0 = 0, x0 = 0, h = H, w = W;
  for (int64_t i = 0; i < H * W; ++i)
    if (dirs[i] != OR_NODATA && !(alpha[i] >= 0.0f && alpha[i] <= 1.0f)) return 1;
  const int64_t N = h * w;
  for (int64_t i = 0; i < N; ++i)
    if (dirs[i] > 8 && dirs[i] != OR_NODATA) return 2;
  uint8_t* D = (uint8_t*)calloc((size_t)N, 1);
  if (!D) return 5;
  int64_t ndata = 0;
  for (int64_t yy = y0; yy < y0 + h; ++yy)
    for (int64_t xx = x0; xx < x0 + w; ++xx) {
      int64_t i = yy * W + xx;
      if (dirs[i] == OR_NODATA) continue;
      ++ndata;
      int64_t t = o_target(dirs, W, xx, yy, y0, x0, h, w);
      if (t >= 0) D[t]++;
    }
  for (int64_t i = 0; i < N; ++i) A[i] = dirs[i] == OR_NODATA ? NAN : (wt ? (double)wt[i] : 1.0);
  int64_t retired = 0;
  for (int64_t q = 0; q < N; ++q) {
    if (dirs[q] == OR_NODATA || D[q] != 0) continue;
    int64_t c = q;
    for (;;) {
      D[c] = 255;
      ++retired;
      int64_t t = o_target(dirs, W, c % W, c / W, y0, x0, h, w);
      if (t < 0) break;
      A[t] += (double)alpha[c] * A[c];
      if (--D[t] > 0) break;
      c = t;
    }
  }
  free(D);
  return retired == ndata ? 0 : 3;
}

/* O-BRUTE with absorption: Eq. 1 unrolled -- every data cell q sends w(q)
 * down its path, scaled by alpha of every cell it leaves:
 *   A(p) = sum_{q upstream of p (or p)} w(q) prod_{u on q..p, u != p} alpha(u).
 * Independent of Kahn; small rasters only. */
int or_brute_alpha_f64(const uint8_t* dirs, int64_t H, int64_t W, const float* wt, const float* alpha,
                       double* A) {
  const int64_t N = H * W;
  for (int64_t i = 0; i < N; ++i) {
    if (dirs[i] > 8 && dirs[i] != OR_NODATA) return 2;
    A[i] = dirs[i] == OR_NODATA ? NAN : 0.0;
  }
  for (int64_t q = 0; q < N; ++q) {
    if (dirs[q] == OR_NODATA) continue;
    double v = wt ? (double)wt[q] : 1.0;
    int64_t c = q, steps = 0;
    while (c >= 0) {
      A[c] += v;
      if (++steps > N) return 3;
      v *= (double)alpha[c];
      c = o_target(dirs, W, c % W, c / W, 0, 0, H, W);
    }
  }
  return 0;
}

/* ======================================================================
 * O-FILL ("the depressions can be filled to the level of
 * their lowest outlets ... Priority-Flood", D15): Priority-Flood + epsilon,
 * literally.  Seeds (data cells on the grid edge or 8-adjacent to NoData)
 * enter a min-priority queue keyed (W, linear index) with W = z; popping a
 * cell c closes each unvisited data neighbour n with
 * W(n) = max(z(n), nextafterf(W(c), +inf)) and pushes it.  NoData (z ==
 * nodata or non-finite) is copied unchanged.  Plain binary heap of
 * (value, index) pairs compared as floats; single-threaded.
 * ==================================================================== */
typedef struct {
  float v;
  int64_t i;
} o_item;
static int o_less(o_item a, o_item b) { return a.v < b.v || (a.v == b.v && a.i < b.i); }

int or_fill(const float* z, int64_t H, int64_t W, float nodata, float* out) {
  const int64_t N = H * W;
  o_item* heap = (o_item*)malloc((size_t)N * sizeof(o_item));
  uint8_t* seen = (uint8_t*)calloc((size_t)N, 1);
  if (!heap || !seen) { free(heap); free(seen); return 5; }
  int64_t hn = 0;
  for (int64_t i = 0; i < N; ++i) out[i] = z[i];
  for (int64_t y = 0; y < H; ++y)
    for (int64_t x = 0; x < W; ++x) {
      const int64_t i = y * W + x;
      if (o_is_nodata(z[i], nodata)) continue;
      int seed = (y == 0 || x == 0 || y == H - 1 || x == W - 1);
      for (int k = 1; k <= 8 && !seed; ++k) {
        const int64_t ny = y + ODY[k], nx = x + ODX[k];
        if (o_is_nodata(z[ny * W + nx], nodata)) seed = 1;
      }
      if (!seed) continue;
      seen[i] = 1;
      /* push */
      o_item it = {z[i], i};
      int64_t c = hn++;
      while (c > 0) {
        int64_t p = (c - 1) / 2;
        if (!o_less(it, heap[p])) break;
        heap[c] = heap[p];
        c = p;
      }
      heap[c] = it;
    }
  while (hn > 0) {
    o_item top = heap[0];
    o_item last = heap[--hn];
    int64_t c = 0;
    for (;;) { /* sift down */
      int64_t l = 2 * c + 1;
      if (l >= hn) break;
      int64_t r = l + 1, m = (r < hn && o_less(heap[r], heap[l])) ? r : l;
      if (!o_less(heap[m], last)) break;
      heap[c] = heap[m];
      c = m;
    }
    if (hn > 0) heap[c] = last;
    const int64_t y = top.i / W, x = top.i % W;
    for (int k = 1; k <= 8; ++k) {
      const int64_t ny = y + ODY[k], nx = x + ODX[k];
      if (ny < 0 || nx < 0 || ny >= H || nx >= W) continue;
      const int64_t n = ny * W + nx;
      if (seen[n] || o_is_nodata(z[n], nodata)) continue;
      seen[n] = 1;
      const float up = nextafterf(top.v, INFINITY);
      out[n] = z[n] > up ? z[n] : up;
      o_item it = {out[n], n};
      int64_t cc = hn++;
      while (cc > 0) {
        int64_t p = (cc - 1) / 2;
        if (!o_less(it, heap[p])) break;
        heap[cc] = heap[p];
        cc = p;
      }
      heap[cc] = it;
    }
  }
  free(heap);
  free(seen);
  return 0;
}

int or_acc_u64(const uint8_t* dirs, int64_t H, int64_t W, const uint32_t* wt, uint64_t* A) {
  return or_acc_region_u64(dirs, H, W, 0, 0, H, W, wt, A);
}
int or_acc_f64(const uint8_t* dirs, int64_t H, int64_t W, const float* wt, double* A) {
  return or_acc_region_f64(dirs, H, W, 0, 0, H, W, wt, A);
}

/* ======================================================================
 * O-BRUTE: Eq. 1 unrolled: every data cell q adds w(q) to itself and to
 * every cell on its downstream path (the definition of "flow passing
 * through a cell").  Independent of Kahn; small rasters only.
 * ==================================================================== */
int or_brute_u64(const uint8_t* dirs, int64_t H, int64_t W, const uint32_t* wt, uint64_t* A) {
  const int64_t N = H * W;
  for (int64_t i = 0; i < N; ++i) {
    if (dirs[i] > 8 && dirs[i] != OR_NODATA) return 2;
    A[i] = dirs[i] == OR_NODATA ? UINT64_MAX : 0;
  }
  for (int64_t q = 0; q < N; ++q) {
    if (dirs[q] == OR_NODATA) continue;
    uint64_t wq = wt ? wt[q] : 1;
    int64_t c = q, steps = 0;
    while (c >= 0) {
      A[c] += wq;
      if (++steps > N) return 3;
      c = o_target(dirs, W, c % W, c / W, 0, 0, H, W);
    }
  }
  return 0;
}

/* ======================================================================
 * Perimeter indexing: clockwise from (0,0): top row left->right
 * (0..w-1), right column (w..w+h-2), bottom row right-1 -> left, left column
 * bottom-1 -> top+1.  Degenerate h==1 or w==1: row-major over all cells.
 * P = 2w + 2h - 4.
 * ==================================================================== */
int64_t or_perim_count(int64_t h, int64_t w) {
  if (h <= 0 || w <= 0) return 0;
  if (h == 1 || w == 1) return h * w;
  return 2 * w + 2 * h - 4;
}

int or_perim_xy(int64_t p, int64_t h, int64_t w, int64_t* x, int64_t* y) {
  int64_t P = or_perim_count(h, w);
  if (p < 0 || p >= P) return 1;
  if (h == 1 || w == 1) {
    *y = p / w;
    *x = p % w;
    return 0;
  }
  if (p < w) { *x = p; *y = 0; return 0; }
  p -= w;
  if (p < h - 1) { *x = w - 1; *y = p + 1; return 0; }
  p -= h - 1;
  if (p < w - 1) { *x = w - 2 - p; *y = h - 1; return 0; }
  p -= w - 1;
  *x = 0;
  *y = h - 2 - p;
  return 0;
}

int64_t or_perim_index(int64_t x, int64_t y, int64_t h, int64_t w) {
  if (x < 0 || y < 0 || x >= w || y >= h) return -1;
  if (h == 1 || w == 1) return y * w + x;
  if (y == 0) return x;
  if (x == w - 1) return w + y - 1;
  if (y == h - 1) return w + (h - 1) + (w - 2 - x);
  if (x == 0) return w + (h - 1) + (w - 1) + (h - 2 - y);
  return -1; /* interior */
}

/* tile layout (D20): tiles of th x tw, ragged in the last tile row/column.
 * Tile t = ty*TC + tx; perimeter slots of tile t start at base[t]. */
static void o_tile_geom(int64_t H, int64_t W, int64_t th, int64_t tw, int64_t t, int64_t* y0,
                        int64_t* x0, int64_t* h, int64_t* w) {
  int64_t TC = (W + tw - 1) / tw;
  int64_t ty = t / TC, tx = t % TC;
  *y0 = ty * th;
  *x0 = tx * tw;
  *h = (*y0 + th <= H) ? th : H - *y0;
  *w = (*x0 + tw <= W) ? tw : W - *x0;
}

int64_t or_tiles_perim_total(int64_t H, int64_t W, int64_t th, int64_t tw, int64_t* base) {
  int64_t TR = (H + th - 1) / th, TC = (W + tw - 1) / tw, tot = 0;
  for (int64_t t = 0; t < TR * TC; ++t) {
    int64_t y0, x0, h, w;
    o_tile_geom(H, W, th, tw, t, &y0, &x0, &h, &w);
    if (base) base[t] = tot;
    tot += or_perim_count(h, w);
  }
  if (base) base[TR * TC] = tot;
  return tot;
}

/* ======================================================================
 * O-TILE pieces (intermediate pins P7).
 * A_T: Alg. 1 per tile = or_acc_region_* on each tile.
 * L  : Alg. 2 FollowPath, literally.
 * x  : offsets x(v) = sum_{n not in T, target(n)=v} A_global(n)  (D11).
 * ==================================================================== */
/* Alg. 2 for perimeter cell (cx,cy) of the tile [y0,y0+h)x[x0,x0+w). */
static uint32_t o_follow_path(const uint8_t* dirs, int64_t H, int64_t W, int64_t y0, int64_t x0,
                              int64_t h, int64_t w, int64_t cx, int64_t cy) {
  const int64_t c0x = cx, c0y = cy;
  int64_t steps = 0;
  for (;;) {
    uint8_t f = dirs[cy * W + cx];
    if (f == OR_NODATA || f == OR_NOFLOW) return OR_FLOW_TERMINATES;
    int64_t nx = cx + ODX[f], ny = cy + ODY[f];
    int outside_tile = nx < x0 || ny < y0 || nx >= x0 + w || ny >= y0 + h;
    (void)H;
    if (outside_tile) {
      if (cx == c0x && cy == c0y) return OR_FLOW_EXTERNAL;
      return (uint32_t)or_perim_index(cx - x0, cy - y0, h, w);
    }
    cx = nx;
    cy = ny;
    if (++steps > h * w) return OR_LINK_CYCLE; /* cycle (never a valid index) */
  }
}

int or_links(const uint8_t* dirs, int64_t H, int64_t W, int64_t th, int64_t tw, uint32_t* L) {
  int64_t TR = (H + th - 1) / th, TC = (W + tw - 1) / tw, s = 0;
  for (int64_t t = 0; t < TR * TC; ++t) {
    int64_t y0, x0, h, w;
    o_tile_geom(H, W, th, tw, t, &y0, &x0, &h, &w);
    int64_t P = or_perim_count(h, w);
    for (int64_t p = 0; p < P; ++p) {
      int64_t px, py;
      or_perim_xy(p, h, w, &px, &py);
      L[s++] = o_follow_path(dirs, H, W, y0, x0, h, w, x0 + px, y0 + py);
    }
  }
  return 0;
}

/* per-slot dirs and A_T (tile-local accumulation), u64 / f64 */
int or_tile_acc_u64(const uint8_t* dirs, int64_t H, int64_t W, int64_t th, int64_t tw,
                    const uint32_t* wt, uint64_t* AT) {
  int64_t TR = (H + th - 1) / th, TC = (W + tw - 1) / tw;
  for (int64_t t = 0; t < TR * TC; ++t) {
    int64_t y0, x0, h, w;
    o_tile_geom(H, W, th, tw, t, &y0, &x0, &h, &w);
    int rc = or_acc_region_u64(dirs, H, W, y0, x0, h, w, wt, AT);
    if (rc) return rc;
  }
  return 0;
}
int or_tile_acc_f64(const uint8_t* dirs, int64_t H, int64_t W, int64_t th, int64_t tw,
                    const float* wt, double* AT) {
  int64_t TR = (H + th - 1) / th, TC = (W + tw - 1) / tw;
  for (int64_t t = 0; t < TR * TC; ++t) {
    int64_t y0, x0, h, w;
    o_tile_geom(H, W, th, tw, t, &y0, &x0, &h, &w);
    int rc = or_acc_region_f64(dirs, H, W, y0, x0, h, w, wt, AT);
    if (rc) return rc;
  }
  return 0;
}

/* x(v) per perimeter slot from a global accumulation (u64 / f64) */
int or_offsets_u64(const uint8_t* dirs, int64_t H, int64_t W, int64_t th, int64_t tw,
                   const uint64_t* A, uint64_t* X) {
  int64_t TR = (H + th - 1) / th, TC = (W + tw - 1) / tw, s = 0;
  for (int64_t t = 0; t < TR * TC; ++t) {
    int64_t y0, x0, h, w;
    o_tile_geom(H, W, th, tw, t, &y0, &x0, &h, &w);
    int64_t P = or_perim_count(h, w);
    for (int64_t p = 0; p < P; ++p, ++s) {
      int64_t px, py;
      or_perim_xy(p, h, w, &px, &py);
      int64_t vx = x0 + px, vy = y0 + py;
      uint64_t acc = 0;
      if (dirs[vy * W + vx] != OR_NODATA) {
        for (int k = 1; k <= 8; ++k) { /* neighbour n = v - offset(k'), look at all 8 */
          int64_t nx = vx + ODX[k], ny = vy + ODY[k];
          if (nx < 0 || ny < 0 || nx >= W || ny >= H) continue;
          if (nx >= x0 && ny >= y0 && nx < x0 + w && ny < y0 + h) continue; /* in tile */
          if (o_target(dirs, W, nx, ny, 0, 0, H, W) == vy * W + vx) acc += A[ny * W + nx];
        }
      }
      X[s] = acc;
    }
  }
  return 0;
}
int or_offsets_f64(const uint8_t* dirs, int64_t H, int64_t W, int64_t th, int64_t tw,
                   const double* A, double* X) {
  int64_t TR = (H + th - 1) / th, TC = (W + tw - 1) / tw, s = 0;
  for (int64_t t = 0; t < TR * TC; ++t) {
    int64_t y0, x0, h, w;
    o_tile_geom(H, W, th, tw, t, &y0, &x0, &h, &w);
    int64_t P = or_perim_count(h, w);
    for (int64_t p = 0; p < P; ++p, ++s) {
      int64_t px, py;
      or_perim_xy(p, h, w, &px, &py);
      int64_t vx = x0 + px, vy = y0 + py;
      double acc = 0.0;
      if (dirs[vy * W + vx] != OR_NODATA) {
        for (int k = 1; k <= 8; ++k) {
          int64_t nx = vx + ODX[k], ny = vy + ODY[k];
          if (nx < 0 || ny < 0 || nx >= W || ny >= H) continue;
          if (nx >= x0 && ny >= y0 && nx < x0 + w && ny < y0 + h) continue;
          if (o_target(dirs, W, nx, ny, 0, 0, H, W) == vy * W + vx) acc += A[ny * W + nx];
        }
      }
      X[s] = acc;
    }
  }
  return 0;
}

/* ======================================================================
 * O-PAPER: a literal single-threaded rendition of the paper's tiled method
 * (u64 and f64 accumulators):
 *   stage 1, per tile: Alg. 1 with a FIFO queue, then Alg. 2
 *     for every perimeter cell; payload F, A, L
 *     per perimeter cell;
 *   stage 2, producer: global flow graph over all perimeter cells, joining
 *     adjoining edges and corners; solved with "the same strategy"
 *     as Alg. 1 with the two modifications of P:L217-222: non-FlowExternal
 *     cells start at A=0, and additions are tracked in an offset array A'
 *     which is split into a_in (external inflow, returned to the tile) and
 *     a_int (internal-link inflow) (D11);
 *   stage 3, per tile: EVICT -- rerun Alg. 1 and add a_in to
 *     every downstream in-tile cell of each perimeter cell's flow path
 *     ("add A' to every cell in its downstream flow path").
 * ==================================================================== */
#define OR_PAPER_BODY(T, WEXPR, NDMARK, ACCFN)                                              \
  if (H <= 0 || W <= 0 || th <= 0 || tw <= 0) return 1;                                  \
  if (or_validate(dirs, H * W) >= 0) return 2;                                           \
  const int64_t TR = (H + th - 1) / th, TC = (W + tw - 1) / tw, NT = TR * TC;            \
  int64_t* base = (int64_t*)malloc((size_t)(NT + 1) * sizeof(int64_t));                  \
  const int64_t NP = or_tiles_perim_total(H, W, th, tw, base);                          \
  T* pA = (T*)malloc((size_t)NP * sizeof(T));                                            \
  uint32_t* pL = (uint32_t*)malloc((size_t)NP * sizeof(uint32_t));                       \
  uint8_t* pF = (uint8_t*)malloc((size_t)NP);                                            \
  T* a_in = (T*)calloc((size_t)NP, sizeof(T));                                           \
  T* a_int = (T*)calloc((size_t)NP, sizeof(T));                                          \
  T* gA = (T*)malloc((size_t)NP * sizeof(T));                                            \
  int64_t* nxt = (int64_t*)malloc((size_t)NP * sizeof(int64_t));                         \
  int* ext = (int*)malloc((size_t)NP * sizeof(int));                                     \
  uint32_t* indeg = (uint32_t*)calloc((size_t)NP, sizeof(uint32_t));                     \
  int64_t* q = (int64_t*)malloc((size_t)(NP > 0 ? NP : 1) * sizeof(int64_t));            \
  int rc = 0;                                                                            \
  /* ---- stage 1: Alg. 1 + Alg. 2 per tile, payload per perimeter cell ---- */         \
  for (int64_t t = 0; t < NT && !rc; ++t) {                                              \
    int64_t y0, x0, h, w;                                                                \
    o_tile_geom(H, W, th, tw, t, &y0, &x0, &h, &w);                                      \
    rc = ACCFN(dirs, H, W, y0, x0, h, w, wt, A, 1);                                      \
    int64_t P = or_perim_count(h, w);                                                    \
    for (int64_t p = 0; p < P; ++p) {                                                    \
      int64_t px, py;                                                                    \
      or_perim_xy(p, h, w, &px, &py);                                                    \
      int64_t i = (y0 + py) * W + x0 + px;                                               \
      pF[base[t] + p] = dirs[i];                                                         \
      pA[base[t] + p] = A[i];                                                            \
      pL[base[t] + p] = o_follow_path(dirs, H, W, y0, x0, h, w, x0 + px, y0 + py);       \
    }                                                                                    \
  }                                                                                      \
  /* ---- stage 2: producer builds and solves the global flow graph ---- */             \
  for (int64_t t = 0; t < NT && !rc; ++t) {                                              \
    int64_t y0, x0, h, w;                                                                \
    o_tile_geom(H, W, th, tw, t, &y0, &x0, &h, &w);                                      \
    int64_t P = or_perim_count(h, w);                                                    \
    for (int64_t p = 0; p < P; ++p) {                                                    \
      int64_t s = base[t] + p;                                                           \
      nxt[s] = -1;                                                                       \
      ext[s] = 0;                                                                        \
      /* modification 1: cells not FlowExternal start at A = 0 */              \
      gA[s] = pL[s] == OR_FLOW_EXTERNAL ? pA[s] : (T)0;                                  \
      if (pL[s] == OR_FLOW_EXTERNAL) {                                                   \
        int64_t px, py;                                                                  \
        or_perim_xy(p, h, w, &px, &py);                                                  \
        int64_t nx = x0 + px + ODX[pF[s]], ny = y0 + py + ODY[pF[s]];                    \
        /* edge to the adjoining tile's perimeter cell (edges or corners,                \
         * P:L215); dropped when the target is off the DEM or NoData (D22) */          \
        if (nx >= 0 && ny >= 0 && nx < W && ny < H && dirs[ny * W + nx] != OR_NODATA) {  \
          int64_t t2 = (ny / th) * TC + nx / tw, y2, x2, h2, w2;                         \
          o_tile_geom(H, W, th, tw, t2, &y2, &x2, &h2, &w2);                             \
          nxt[s] = base[t2] + or_perim_index(nx - x2, ny - y2, h2, w2);                  \
          ext[s] = 1;                                                                    \
        }                                                                                \
      } else if (pL[s] != OR_FLOW_TERMINATES) {                                          \
        if (pL[s] >= (uint32_t)P) rc = 3;                                                \
        else nxt[s] = base[t] + pL[s];                                                   \
      }                                                                                  \
      if (nxt[s] >= 0) indeg[nxt[s]]++;                                                  \
    }                                                                                    \
  }                                                                                      \
  int64_t qh = 0, qt = 0, done = 0;                                                      \
  for (int64_t s = 0; s < NP && !rc; ++s)                                                \
    if (indeg[s] == 0) q[qt++] = s;                                                      \
  while (qh < qt && !rc) {                                                               \
    int64_t s = q[qh++];                                                                 \
    ++done;                                                                              \
    if (nxt[s] < 0) continue;                                                            \
    /* modification 2: pass A + A' downstream */                               \
    T out = gA[s] + a_in[s] + a_int[s];                                                  \
    if (ext[s]) a_in[nxt[s]] += out;                                                     \
    else a_int[nxt[s]] += out;                                                           \
    if (--indeg[nxt[s]] == 0) q[qt++] = nxt[s];                                          \
  }                                                                                      \
  if (!rc && done != NP) rc = 3;                                                         \
  /* ---- stage 3: EVICT: rerun Alg. 1, add a_in down each path ---- */                 \
  for (int64_t t = 0; t < NT && !rc; ++t) {                                              \
    int64_t y0, x0, h, w;                                                                \
    o_tile_geom(H, W, th, tw, t, &y0, &x0, &h, &w);                                      \
    rc = ACCFN(dirs, H, W, y0, x0, h, w, wt, A, 1);                                      \
    int64_t P = or_perim_count(h, w);                                                    \
    for (int64_t p = 0; p < P && !rc; ++p) {                                             \
      T off = a_in[base[t] + p];                                                         \
      if (off == (T)0) continue;                                                         \
      int64_t px, py;                                                                    \
      or_perim_xy(p, h, w, &px, &py);                                                    \
      int64_t cx = x0 + px, cy = y0 + py, steps = 0;                                     \
      for (;;) {                                                                         \
        uint8_t f = dirs[cy * W + cx];                                                   \
        if (f == OR_NODATA) break;                                                       \
        A[cy * W + cx] += off;                                                           \
        if (f == OR_NOFLOW) break;                                                       \
        int64_t nx = cx + ODX[f], ny = cy + ODY[f];                                      \
        if (nx < x0 || ny < y0 || nx >= x0 + w || ny >= y0 + h) break;                   \
        cx = nx;                                                                         \
        cy = ny;                                                                         \
        if (++steps > h * w) { rc = 3; break; }                                          \
      }                                                                                  \
    }                                                                                    \
  }                                                                                      \
  free(base); free(pA); free(pL); free(pF); free(a_in); free(a_int); free(gA);           \
  free(nxt); free(ext); free(indeg); free(q);                                            \
  return rc;

/* Alg. 1 with a FIFO queue on one tile; writes A for the tile. */
#define OR_ALG1_BODY(T, WEXPR, NDMARK)                                                   \
  (void)H;                                                                              \
  const int64_t N = h * w;                                                              \
  uint8_t* D = (uint8_t*)calloc((size_t)N, 1);                                          \
  int64_t* Q = (int64_t*)malloc((size_t)N * sizeof(int64_t));                           \
  if (!D || !Q) { free(D); free(Q); return 5; }                                         \
  /* "Set D(c)=0, A(c)=0 for all c"; first loop */                        \
  for (int64_t yy = y0; yy < y0 + h; ++yy)                                              \
    for (int64_t xx = x0; xx < x0 + w; ++xx) {                                          \
      int64_t i = yy * W + xx;                                                          \
      if (dirs[i] == OR_NODATA) { A[i] = (NDMARK); continue; }                          \
      A[i] = (T)0;                                                                      \
      int64_t t = o_target(dirs, W, xx, yy, y0, x0, h, w);                              \
      if (t >= 0) D[((t / W) - y0) * w + (t % W) - x0]++;                              \
    }                                                                                   \
  /* seed Q with D=0 data cells */                                        \
  int64_t qh = 0, qt = 0;                                                               \
  for (int64_t yy = y0; yy < y0 + h; ++yy)                                              \
    for (int64_t xx = x0; xx < x0 + w; ++xx)                                            \
      if (D[(yy - y0) * w + xx - x0] == 0 && dirs[yy * W + xx] != OR_NODATA)            \
        Q[qt++] = yy * W + xx;                                                          \
  /* queue loop: A(c) += w(c); pass downstream */                         \
  while (qh < qt) {                                                                     \
    int64_t i = Q[qh++];                                                                \
    A[i] += (WEXPR);                                                                    \
    int64_t t = o_target(dirs, W, i % W, i / W, y0, x0, h, w);                          \
    if (t < 0) continue;                                                                \
    A[t] += A[i];                                                                       \
    int64_t tl = ((t / W) - y0) * w + (t % W) - x0;                                     \
    if (--D[tl] == 0) Q[qt++] = t;                                                      \
  }                                                                                     \
  int64_t nd = 0;                                                                       \
  for (int64_t yy = y0; yy < y0 + h; ++yy)                                              \
    for (int64_t xx = x0; xx < x0 + w; ++xx) nd += dirs[yy * W + xx] != OR_NODATA;      \
  free(D); free(Q);                                                                     \
  return qt == nd ? 0 : 3;

static int o_alg1_u64(const uint8_t* dirs, int64_t H, int64_t W, int64_t y0, int64_t x0, int64_t h,
                      int64_t w, const uint32_t* wt, uint64_t* A, int unused) {
  (void)unused;
  OR_ALG1_BODY(uint64_t, (wt ? (uint64_t)wt[i] : (uint64_t)1), UINT64_MAX)
}
static int o_alg1_f64(const uint8_t* dirs, int64_t H, int64_t W, int64_t y0, int64_t x0, int64_t h,
                      int64_t w, const float* wt, double* A, int unused) {
  (void)unused;
  OR_ALG1_BODY(double, (wt ? (double)wt[i] : 1.0), NAN)
}

int or_paper_u64(const uint8_t* dirs, int64_t H, int64_t W, int64_t th, int64_t tw,
                 const uint32_t* wt, uint64_t* A){OR_PAPER_BODY(uint64_t, 0, 0, o_alg1_u64)}

int or_paper_f64(const uint8_t* dirs, int64_t H, int64_t W, int64_t th, int64_t tw,
                 const float* wt, double* A){OR_PAPER_BODY(double, 0, 0, o_alg1_f64)}

/* ======================================================================
 * Certificates and workload statistics (pins P8; DESIGN.md workload
 * characterisation).
 * ==================================================================== */
/* Donor identity A(p) - w(p) == sum_{target(n)=p} A(n) at every data cell,
 * NoData marker at NoData cells, and sum over terminal cells (no target:
 * outlets off-grid / into NoData, NoFlow) == sum w.  Exact, u64.
 * Returns the number of violating cells (+1 if the mass balance fails). */
int64_t or_certify_u64(const uint8_t* dirs, int64_t H, int64_t W, const uint32_t* wt,
                       const uint64_t* A) {
  int64_t bad = 0;
  uint64_t sw = 0, so = 0;
  for (int64_t y = 0; y < H; ++y)
    for (int64_t x = 0; x < W; ++x) {
      int64_t i = y * W + x;
      if (dirs[i] == OR_NODATA) {
        bad += A[i] != UINT64_MAX;
        continue;
      }
      uint64_t wi = wt ? wt[i] : 1, s = 0;
      sw += wi;
      for (int k = 1; k <= 8; ++k) {
        int64_t nx = x + ODX[k], ny = y + ODY[k];
        if (nx < 0 || ny < 0 || nx >= W || ny >= H) continue;
        if (o_target(dirs, W, nx, ny, 0, 0, H, W) == i) s += A[ny * W + nx];
      }
      bad += A[i] != wi + s;
      if (o_target(dirs, W, x, y, 0, 0, H, W) < 0) so += A[i];
    }
  return bad + (so != sw);
}

/* Streamed form of or_certify_u64 (P8), for rasters too large for one host
 * buffer: the caller passes a window of nb rows (a strip plus the halo rows
 * that exist: the row above it unless it starts the raster, the row below it
 * unless it ends it) and checks rows [c0, c1) of the window.  Rows outside
 * the window are off the raster for this check, which is exact because the
 * window holds every row a checked cell's donors or target can lie in.
 * Adds the checked cells' sum w to acc[0] and the sum of A over the checked
 * terminal cells to acc[1]; the caller compares the totals after the last
 * strip (mass balance).  Returns the number of violating cells.           */
int64_t or_certify_rows_u64(const uint8_t* dirs, int64_t nb, int64_t W, const uint32_t* wt,
                            const uint64_t* A, int64_t c0, int64_t c1, uint64_t* acc) {
  int64_t bad = 0;
  for (int64_t y = c0; y < c1; ++y)
    for (int64_t x = 0; x < W; ++x) {
      int64_t i = y * W + x;
      if (dirs[i] == OR_NODATA) {
        bad += A[i] != UINT64_MAX;
        continue;
      }
      uint64_t wi = wt ? wt[i] : 1, s = 0;
      acc[0] += wi;
      for (int k = 1; k <= 8; ++k) {
        int64_t nx = x + ODX[k], ny = y + ODY[k];
        if (nx < 0 || ny < 0 || nx >= W || ny >= nb) continue;
        if (o_target(dirs, W, nx, ny, 0, 0, nb, W) == i) s += A[ny * W + nx];
      }
      bad += A[i] != wi + s;
      if (o_target(dirs, W, x, y, 0, 0, nb, W) < 0) acc[1] += A[i];
    }
  return bad;
}

/* f64 variant: |A(p) - (w(p) + sum donors)| <= rtol * A(p); returns #bad and
 * the max relative residual in *maxrel. */
int64_t or_certify_f64(const uint8_t* dirs, int64_t H, int64_t W, const float* wt,
                       const double* A, double rtol, double* maxrel) {
  int64_t bad = 0;
  double mr = 0.0;
  for (int64_t y = 0; y < H; ++y)
    for (int64_t x = 0; x < W; ++x) {
      int64_t i = y * W + x;
      if (dirs[i] == OR_NODATA) {
        bad += !isnan(A[i]);
        continue;
      }
      double s = wt ? (double)wt[i] : 1.0;
      for (int k = 1; k <= 8; ++k) {
        int64_t nx = x + ODX[k], ny = y + ODY[k];
        if (nx < 0 || ny < 0 || nx >= W || ny >= H) continue;
        if (o_target(dirs, W, nx, ny, 0, 0, H, W) == i) s += A[ny * W + nx];
      }
      double rel = fabs(A[i] - s) / (fabs(A[i]) > 0 ? fabs(A[i]) : 1.0);
      if (!(rel <= rtol)) ++bad;
      if (rel > mr || isnan(rel)) mr = rel;
    }
  if (maxrel) *maxrel = mr;
  return bad;
}

/* Workload characterisation: heights (longest upstream path, edges) via
 * the same chain-following schedule; histogram of heights clipped to
 * nbins-1; returns max height, and writes #outlets, #noflow, max A (u64,
 * unit weights) to out[0..2].  Cells: whole raster.                      */
int64_t or_stats(const uint8_t* dirs, int64_t H, int64_t W, int64_t* hist, int64_t nbins,
                 int64_t* out) {
  const int64_t N = H * W;
  uint8_t* D = (uint8_t*)calloc((size_t)N, 1);
  uint32_t* ht = (uint32_t*)calloc((size_t)N, sizeof(uint32_t));
  uint64_t* A = (uint64_t*)malloc((size_t)N * sizeof(uint64_t));
  if (!D || !ht || !A) return -1;
  int64_t outlets = 0, noflow = 0, maxh = 0;
  uint64_t maxa = 0;
  for (int64_t i = 0; i < N; ++i) {
    A[i] = 1;
    if (dirs[i] == OR_NODATA) continue;
    int64_t t = o_target(dirs, W, i % W, i / W, 0, 0, H, W);
    if (t >= 0) D[t]++;
    else if (dirs[i] == OR_NOFLOW) ++noflow;
    else ++outlets;
  }
  for (int64_t b = 0; b < nbins; ++b) hist[b] = 0;
  for (int64_t p = 0; p < N; ++p) {
    if (dirs[p] == OR_NODATA || D[p] != 0) continue;
    int64_t c = p;
    for (;;) {
      D[c] = 255;
      int64_t hb = ht[c] < (uint32_t)(nbins - 1) ? ht[c] : nbins - 1;
      hist[hb]++;
      if ((int64_t)ht[c] > maxh) maxh = ht[c];
      if (A[c] > maxa) maxa = A[c];
      int64_t t = o_target(dirs, W, c % W, c / W, 0, 0, H, W);
      if (t < 0) break;
      A[t] += A[c];
      if (ht[c] + 1 > ht[t]) ht[t] = ht[c] + 1;
      if (--D[t] > 0) break;
      c = t;
    }
  }
  out[0] = outlets;
  out[1] = noflow;
  out[2] = (int64_t)maxa;
  free(D);
  free(ht);
  free(A);
  return maxh;
}
