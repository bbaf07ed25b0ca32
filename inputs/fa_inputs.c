/*
 * fa_inputs.c -- seeded synthetic input generators shared by the oracle
 * tests and the CUDA path (tests + bench).  Recipes G1..G6 of DESIGN.md
 * section "Input recipe".
 *
 * This module holds NONE of the method's arithmetic: no D8 rule, no
 * accumulation, no tiling.  It only produces elevation rasters, weights
 * and direction rasters with a known closed-form structure.  It is built
 * with -ffp-contract=off and without -ffast-math so that every box
 * regenerates bit-identical inputs (generation is counter-based, so the
 * OpenMP schedule cannot change a value).
 *
 * Stand-in for the paper's SRTM / NED / PAMAP rasters (Table 1,
 * L372-391), which are not available: fractal relief, depression-filled
 * ("filled"), irregular NoData coast (L407, L416).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------- G1: counter-based RNG ---------------- */
static inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
/* u(seed, stream, i) in [0,1) with 53 random bits */
static inline double g1_u(uint64_t seed, uint64_t stream, uint64_t i) {
  return (double)(splitmix64(seed ^ (stream << 56) ^ i) >> 11) * 0x1.0p-53;
}
double fa_in_u01(uint64_t seed, uint64_t stream, uint64_t i) { return g1_u(seed, stream, i); }
uint64_t fa_in_splitmix64(uint64_t x) { return splitmix64(x); }

static int64_t next_pow2(int64_t v) {
  int64_t n = 1;
  while (n < v) n <<= 1;
  return n;
}

/* ---------------- G2: diamond-square on an n x n torus ----------------
 * v(0,0)=0; for s = n, n/2, ..., 2 with amp = r^{log2(n/s)}:
 *   diamond: v(x+h,y+h) = ((a+b)+(c+d))*0.25 + amp*(2u-1)  (4 corners)
 *   square : v(edge midpoint) = ((l+r)+(u+d))*0.25 + amp*(2u-1) (4 wrapped
 *            neighbours at distance h)
 * u is keyed by the point's linear index y*n+x (stream 0).  Values are
 * computed in double and stored as float.  The H x W raster is the top-left
 * crop of the torus, normalised to exactly [0, 1000]:
 *   z = fl32((v - min) / (max - min) * 1000).                             */
int fa_in_terrain(uint64_t seed, int64_t H, int64_t W, double rough, float* z) {
  if (H <= 0 || W <= 0 || !z) return 1;
  int64_t n = next_pow2(H > W ? H : W);
  if (n < 2) n = 2;
  float* v = z;
  int own = 0;
  if (!(n == H && n == W)) {
    v = (float*)malloc((size_t)n * (size_t)n * sizeof(float));
    if (!v) return 5;
    own = 1;
  }
  const int64_t mask = n - 1;
  v[0] = 0.0f;
  double amp = 1.0;
  for (int64_t s = n; s >= 2; s >>= 1, amp *= rough) {
    const int64_t h = s >> 1;
    const int64_t cnt = n / s;
    /* diamond step: centres of s-squares */
#pragma omp parallel for schedule(static)
    for (int64_t by = 0; by < cnt; ++by) {
      for (int64_t bx = 0; bx < cnt; ++bx) {
        int64_t x = bx * s, y = by * s;
        int64_t x1 = (x + s) & mask, y1 = (y + s) & mask;
        double a = v[y * n + x], b = v[y * n + x1], c = v[y1 * n + x], d = v[y1 * n + x1];
        int64_t cx = x + h, cy = y + h;
        uint64_t idx = (uint64_t)(cy * n + cx);
        double m = ((a + b) + (c + d)) * 0.25;
        v[cy * n + cx] = (float)(m + amp * (2.0 * g1_u(seed, 0, idx) - 1.0));
      }
    }
    /* square step: edge midpoints (x+h, y) and (x, y+h) */
#pragma omp parallel for schedule(static)
    for (int64_t by = 0; by < cnt; ++by) {
      for (int64_t bx = 0; bx < cnt; ++bx) {
        int64_t x = bx * s, y = by * s;
        for (int e = 0; e < 2; ++e) {
          int64_t px = e == 0 ? x + h : x;
          int64_t py = e == 0 ? y : y + h;
          double l = v[py * n + ((px - h) & mask)];
          double r = v[py * n + ((px + h) & mask)];
          double u = v[((py - h) & mask) * n + px];
          double d = v[((py + h) & mask) * n + px];
          uint64_t idx = (uint64_t)(py * n + px);
          double m = ((l + r) + (u + d)) * 0.25;
          v[py * n + px] = (float)(m + amp * (2.0 * g1_u(seed, 0, idx) - 1.0));
        }
      }
    }
  }
  /* crop + normalise */
  double mn = INFINITY, mx = -INFINITY;
#pragma omp parallel for reduction(min : mn) reduction(max : mx) schedule(static)
  for (int64_t y = 0; y < H; ++y)
    for (int64_t x = 0; x < W; ++x) {
      double t = v[y * n + x];
      if (t < mn) mn = t;
      if (t > mx) mx = t;
    }
  double span = mx - mn;
  if (own) {
    for (int64_t y = 0; y < H; ++y)
      for (int64_t x = 0; x < W; ++x) {
        double t = v[y * n + x];
        z[y * W + x] = span > 0 ? (float)((t - mn) / span * 1000.0) : 0.0f;
      }
    free(v);
  } else {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < H * W; ++i) {
      double t = z[i];
      z[i] = span > 0 ? (float)((t - mn) / span * 1000.0) : 0.0f;
    }
  }
  return 0;
}

/* ---------------- G3: NoData coast ----------------
 * 1-D midpoint displacement on a ring of m = 2^k >= H points (stream 1,
 * multiplier r per octave), crop to H rows, normalise to [-1,1]:
 *   c(y) = clamp(round(f*W*(1 + 0.5*(p(y) - mean p))), 1, W-1)
 * cell (x,y) is NoData (z = nodata) iff x < c(y).  The region contains the
 * whole west column, so it is connected and touches the west edge.
 * Returns the number of NoData cells written (or -1 on error).           */
int64_t fa_in_coast(uint64_t seed, int64_t H, int64_t W, double frac, double rough,
                    float nodata, float* z) {
  if (H <= 0 || W < 2 || !z || frac <= 0) return frac <= 0 ? 0 : -1;
  int64_t m = next_pow2(H);
  if (m < 2) m = 2;
  double* p = (double*)malloc((size_t)m * sizeof(double));
  if (!p) return -1;
  p[0] = 0.0;
  double amp = 1.0;
  for (int64_t s = m; s >= 2; s >>= 1, amp *= rough) {
    int64_t h = s >> 1;
    for (int64_t i = 0; i < m; i += s) {
      double a = p[i], b = p[(i + s) & (m - 1)];
      p[i + h] = (a + b) * 0.5 + amp * (2.0 * g1_u(seed, 1, (uint64_t)(i + h)) - 1.0);
    }
  }
  double mn = INFINITY, mx = -INFINITY, mean = 0.0;
  for (int64_t y = 0; y < H; ++y) {
    if (p[y] < mn) mn = p[y];
    if (p[y] > mx) mx = p[y];
  }
  double span = mx - mn;
  for (int64_t y = 0; y < H; ++y) {
    p[y] = span > 0 ? 2.0 * (p[y] - mn) / span - 1.0 : 0.0;
    mean += p[y];
  }
  mean /= (double)H;
  int64_t total = 0;
#pragma omp parallel for reduction(+ : total) schedule(static)
  for (int64_t y = 0; y < H; ++y) {
    double cf = frac * (double)W * (1.0 + 0.5 * (p[y] - mean));
    int64_t c = llround(cf);
    if (c < 1) c = 1;
    if (c > W - 1) c = W - 1;
    for (int64_t x = 0; x < c; ++x) z[y * W + x] = nodata;
    total += c;
  }
  free(p);
  return total;
}

/* ---------------- G4: depression filling (Priority-Flood + epsilon) -------
 * PAPER.md L59 fills depressions with the Priority-Flood (Barnes et al.
 * 2014).  Its epsilon variant is the Dijkstra-style flood whose result we
 * define exactly as the least epsilon-cost surface W:
 *   seeds S = data cells on the grid edge or 8-adjacent to NoData
 *   W(s) = z(s)                                   for s in S
 *   W(p) = max(z(p), nextafterf(min_{data n in N8(p)} W(n), +inf))  otherwise
 * Every step strictly increases the cost, so W is unique (a shortest-path
 * fixpoint): any correct schedule yields the same bits.  We compute it with
 * a tiled label-correcting Dijkstra (OpenMP over tiles, synchronous rounds,
 * a binary heap per tile); the single-tile run is plain Dijkstra = the
 * classic Priority-Flood order.  Every non-seed data cell ends strictly above
 * its minimising neighbour, so D8 on W has no NoFlow cell and every path
 * drains to a seed (pins P14).  NoData cells are never touched.
 * Returns the number of raised cells (W > z), or <0 on error.             */
typedef struct {
  uint64_t* a;
  size_t n, cap;
} u64vec;
static int u64_push(u64vec* v, uint64_t x) {
  if (v->n == v->cap) {
    size_t nc = v->cap ? v->cap * 2 : 64;
    uint64_t* na = (uint64_t*)realloc(v->a, nc * sizeof(uint64_t));
    if (!na) return 1;
    v->a = na;
    v->cap = nc;
  }
  v->a[v->n++] = x;
  return 0;
}
/* binary min-heap of (key << 32 | local index) */
static void heap_push(u64vec* h, uint64_t x) {
  u64_push(h, x);
  size_t i = h->n - 1;
  uint64_t* a = h->a;
  while (i) {
    size_t p = (i - 1) >> 1;
    if (a[p] <= x) break;
    a[i] = a[p];
    i = p;
  }
  a[i] = x;
}
static uint64_t heap_pop(u64vec* h) {
  uint64_t* a = h->a;
  uint64_t top = a[0];
  uint64_t x = a[--h->n];
  size_t n = h->n, i = 0;
  if (!n) return top;
  for (;;) {
    size_t l = 2 * i + 1;
    if (l >= n) break;
    size_t r = l + 1, m = (r < n && a[r] < a[l]) ? r : l;
    if (a[m] >= x) break;
    a[i] = a[m];
    i = m;
  }
  a[i] = x;
  return top;
}
static inline int is_nd(float v, float nodata) { return !isfinite(v) || v == nodata; }
static inline uint32_t fkey(float f) {
  uint32_t k;
  memcpy(&k, &f, 4);
  return k; /* f >= +0: unsigned order == float order */
}
static inline float kf(uint32_t k) {
  float f;
  memcpy(&f, &k, 4);
  return f;
}

int64_t fa_in_fill_tiled(int64_t H, int64_t W, float nodata, float* z, int64_t tile) {
  static const int DX[8] = {0, 1, 1, 1, 0, -1, -1, -1};
  static const int DY[8] = {-1, -1, 0, 1, 1, 1, 0, -1};
  if (H <= 0 || W <= 0 || !z) return -1;
  if (tile <= 0) tile = H > W ? H : W;
  if (tile > 65535) tile = 65535; /* local index must fit 32 bits */
  const int64_t N = H * W;
  const int64_t TR = (H + tile - 1) / tile, TC = (W + tile - 1) / tile, NT = TR * TC;
  float* Wv = (float*)malloc((size_t)N * sizeof(float));
  uint8_t* pend = (uint8_t*)calloc((size_t)N, 1); /* cell queued for relaxation */
  uint8_t* tile_act = (uint8_t*)calloc((size_t)NT, 1);
  u64vec* outb = (u64vec*)calloc((size_t)NT, sizeof(u64vec)); /* (cand<<32|dummy) pairs */
  u64vec* outi = (u64vec*)calloc((size_t)NT, sizeof(u64vec));
  if (!Wv || !pend || !tile_act || !outb || !outi) return -1;
  int bad = 0;
#pragma omp parallel for reduction(| : bad) schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    float v = z[i];
    if (!is_nd(v, nodata) && (v < 0.0f || signbit(v))) bad = 1;
    Wv[i] = is_nd(v, nodata) ? v : INFINITY;
  }
  if (bad) return -2;
  /* seeds */
#pragma omp parallel for schedule(static)
  for (int64_t y = 0; y < H; ++y)
    for (int64_t x = 0; x < W; ++x) {
      int64_t i = y * W + x;
      if (is_nd(z[i], nodata)) continue;
      int s = (y == 0 || x == 0 || y == H - 1 || x == W - 1);
      for (int k = 0; k < 8 && !s; ++k)
        if (is_nd(z[(y + DY[k]) * W + x + DX[k]], nodata)) s = 1;
      if (s) {
        Wv[i] = z[i];
        pend[i] = 1;
      }
    }
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < NT; ++t) {
    int64_t ty = t / TC, tx = t % TC;
    int64_t y1 = ty * tile + tile < H ? ty * tile + tile : H;
    int64_t x1 = tx * tile + tile < W ? tx * tile + tile : W;
    for (int64_t y = ty * tile; y < y1 && !tile_act[t]; ++y)
      for (int64_t x = tx * tile; x < x1; ++x)
        if (pend[y * W + x]) {
          tile_act[t] = 1;
          break;
        }
  }
  for (;;) {
    int64_t nact = 0;
    for (int64_t t = 0; t < NT; ++t) nact += tile_act[t];
    if (!nact) break;
#pragma omp parallel
    {
      u64vec heap = {0, 0, 0};
#pragma omp for schedule(dynamic, 1)
      for (int64_t t = 0; t < NT; ++t) {
        if (!tile_act[t]) continue;
        tile_act[t] = 0;
        const int64_t ty = t / TC, tx = t % TC;
        const int64_t y0 = ty * tile, x0 = tx * tile;
        const int64_t y1 = y0 + tile < H ? y0 + tile : H;
        const int64_t x1 = x0 + tile < W ? x0 + tile : W;
        const int64_t tw = x1 - x0;
        heap.n = 0;
        for (int64_t y = y0; y < y1; ++y)
          for (int64_t x = x0; x < x1; ++x) {
            int64_t i = y * W + x;
            if (pend[i]) {
              pend[i] = 0;
              heap_push(&heap, ((uint64_t)fkey(Wv[i]) << 32) | (uint64_t)((y - y0) * tw + (x - x0)));
            }
          }
        while (heap.n) {
          uint64_t top = heap_pop(&heap);
          uint32_t key = (uint32_t)(top >> 32), loc = (uint32_t)top;
          int64_t cy = y0 + loc / tw, cx = x0 + loc % tw, c = cy * W + cx;
          if (fkey(Wv[c]) != key) continue; /* stale */
          float nxt = nextafterf(kf(key), INFINITY);
          for (int k = 0; k < 8; ++k) {
            int64_t nx = cx + DX[k], ny = cy + DY[k];
            if (nx < 0 || ny < 0 || nx >= W || ny >= H) continue;
            int64_t n = ny * W + nx;
            float zn = z[n];
            if (is_nd(zn, nodata)) continue;
            float cand = zn > nxt ? zn : nxt;
            if (nx >= x0 && nx < x1 && ny >= y0 && ny < y1) {
              if (cand < Wv[n]) {
                Wv[n] = cand;
                heap_push(&heap, ((uint64_t)fkey(cand) << 32) | (uint64_t)((ny - y0) * tw + (nx - x0)));
              }
            } else {
              u64_push(&outb[t], (uint64_t)fkey(cand));
              u64_push(&outi[t], (uint64_t)n);
            }
          }
        }
      }
      free(heap.a);
    }
    /* apply cross-tile candidates (grouped by destination tile for safety) */
    for (int64_t t = 0; t < NT; ++t) {
      for (size_t j = 0; j < outb[t].n; ++j) {
        int64_t n = (int64_t)outi[t].a[j];
        float cand = kf((uint32_t)outb[t].a[j]);
        if (cand < Wv[n]) {
          Wv[n] = cand;
          pend[n] = 1;
          int64_t ny = n / W, nx = n % W;
          tile_act[(ny / tile) * TC + nx / tile] = 1;
        }
      }
      outb[t].n = outi[t].n = 0;
    }
  }
  int64_t raised = 0;
#pragma omp parallel for reduction(+ : raised) schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    if (!is_nd(z[i], nodata)) {
      if (Wv[i] > z[i]) ++raised;
      z[i] = Wv[i];
    }
  }
  for (int64_t t = 0; t < NT; ++t) {
    free(outb[t].a);
    free(outi[t].a);
  }
  free(outb);
  free(outi);
  free(tile_act);
  free(pend);
  free(Wv);
  return raised;
}

int64_t fa_in_fill(int64_t H, int64_t W, float nodata, float* z) {
  return fa_in_fill_tiled(H, W, nodata, z, 256);
}

/* ---------------- G5: weights ----------------
 * w_i = 0.5f + (float)(splitmix64(seed ^ (2<<56) ^ i) >> 41) * 2^-23,
 * exactly representable, in [0.5, 1.5).                                 */
void fa_in_weights(uint64_t seed, int64_t n, float* w) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    w[i] = 0.5f + (float)(splitmix64(seed ^ (2ULL << 56) ^ (uint64_t)i) >> 41) * 0x1.0p-23f;
}
/* integer weights in [lo, hi] (stream 4) */
void fa_in_weights_u32(uint64_t seed, int64_t n, uint32_t lo, uint32_t hi, uint32_t* w) {
  uint64_t span = (uint64_t)hi - lo + 1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    w[i] = lo + (uint32_t)(splitmix64(seed ^ (4ULL << 56) ^ (uint64_t)i) % span);
}

/* ---------------- G6: serpentine direction rasters ----------------
 * codes: 0 NoFlow, 1 N, 2 NE, 3 E, 4 SE, 5 S, 6 SW, 7 W, 8 NW, 255 NoData
 * Row y flows E if y even, W if odd; the row-end cell flows S.  The last
 * row's end flows S off the grid.  transposed=1 swaps the roles of rows and
 * columns (column x flows S if x even, N if odd; column ends step E).    */
void fa_in_serpentine(int64_t H, int64_t W, int transposed, uint8_t* d) {
#pragma omp parallel for schedule(static)
  for (int64_t y = 0; y < H; ++y)
    for (int64_t x = 0; x < W; ++x) {
      uint8_t c;
      if (!transposed) {
        if (y % 2 == 0) c = (x == W - 1) ? 5 : 3;
        else c = (x == 0) ? 5 : 7;
      } else {
        if (x % 2 == 0) c = (y == H - 1) ? 3 : 5;
        else c = (y == 0) ? 3 : 1;
      }
      d[y * W + x] = c;
    }
}

/* ---------------- random acyclic direction rasters (test fixtures) -------
 * Potential phi(i) = u(seed,3,i) (ties broken by index).  Each cell is
 * NoData with prob p_nodata (stream 5), else NoFlow with prob p_noflow
 * (stream 6), else picks uniformly (stream 7) among
 *   {k : neighbour k off-grid or NoData} U {k : data neighbour with lower
 *   (phi, index)}; NoFlow if that set is empty.
 * Every edge strictly decreases (phi, index), so the raster is acyclic.  */
void fa_in_random_dirs(uint64_t seed, int64_t H, int64_t W, double p_nodata, double p_noflow,
                       uint8_t* d) {
  static const int DX[8] = {0, 1, 1, 1, 0, -1, -1, -1};
  static const int DY[8] = {-1, -1, 0, 1, 1, 1, 0, -1};
  const int64_t N = H * W;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) d[i] = g1_u(seed, 5, (uint64_t)i) < p_nodata ? 255 : 0;
#pragma omp parallel for schedule(static)
  for (int64_t y = 0; y < H; ++y)
    for (int64_t x = 0; x < W; ++x) {
      int64_t i = y * W + x;
      if (d[i] == 255) continue;
      if (g1_u(seed, 6, (uint64_t)i) < p_noflow) {
        d[i] = 0;
        continue;
      }
      double pi = g1_u(seed, 3, (uint64_t)i);
      int cand[8], nc = 0;
      for (int k = 0; k < 8; ++k) {
        int64_t nx = x + DX[k], ny = y + DY[k];
        if (nx < 0 || ny < 0 || nx >= W || ny >= H) {
          cand[nc++] = k;
          continue;
        }
        int64_t n = ny * W + nx;
        if (d[n] == 255) {
          cand[nc++] = k;
          continue;
        }
        double pn = g1_u(seed, 3, (uint64_t)n);
        if (pn < pi || (pn == pi && n < i)) cand[nc++] = k;
      }
      if (nc == 0) {
        d[i] = 0;
        continue;
      }
      int pick = (int)(g1_u(seed, 7, (uint64_t)i) * nc);
      if (pick >= nc) pick = nc - 1;
      d[i] = (uint8_t)(cand[pick] + 1);
    }
}

/* ---------------- quantised random DEM (forces D8 ties) ----------------
 * z = floor(u(seed,8,i) * levels) as float; NoData with prob p_nodata
 * (stream 9) unless p_nodata==0.                                          */
void fa_in_quantized_dem(uint64_t seed, int64_t H, int64_t W, int levels, double p_nodata,
                         float nodata, float* z) {
  const int64_t N = H * W;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    double u = g1_u(seed, 8, (uint64_t)i);
    float v = (float)floor(u * levels);
    if (p_nodata > 0 && g1_u(seed, 9, (uint64_t)i) < p_nodata) v = nodata;
    z[i] = v;
  }
}

int fa_in_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
