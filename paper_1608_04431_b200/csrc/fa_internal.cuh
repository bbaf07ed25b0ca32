// fa_internal.cuh -- shared device/host definitions of libfa (the CUDA path).
// Independent of oracle/: nothing here is shared with the CPU oracle.
//
// Citations: "P:Lnn" = /root/reference/PAPER.md line nn; "Dn" = DESIGN.md reading n.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

// FA_CHECK: device-side bounds / invariant assertions of the checked build
// (tools/build_variant.py checked FA_CHECKED=1, run by tools/check_build.sh);
// compiled out of the product library.  A failed check traps with the file
// and line (cudaErrorAssert), so the checked test run fails loudly.
#ifdef FA_CHECKED
#include <cassert>
#define FA_CHECK(...) assert((__VA_ARGS__))
#else
#define FA_CHECK(...) ((void)0)
#endif

namespace fa {

// ---------------------------------------------------------------- constants
constexpr uint8_t kNoData = 255;  // D1
constexpr uint8_t kNoFlow = 0;
constexpr uint32_t kNone = 0xFFFFFFFFu;            // no node / no parent
constexpr uint32_t kFlowExternal = 0xFFFFFFFEu;    // Alg. 2 sentinel
constexpr uint32_t kFlowTerminates = 0xFFFFFFFFu;  // Alg. 2 sentinel

// Block = the CTA-resident sub-tile: the paper's Alg. 1 + Alg. 2
// run on it entirely in shared memory.  Its shape is a compile-time
// parameter of the block kernels (block.cu) and a run-time field of Geom.
constexpr int kBR = 32;  // default block rows
constexpr int kBC = 32;  // default block cols
#ifndef FA_NW
#define FA_NW 2
#endif
constexpr int kNW = FA_NW;   // warps (one block each) per CTA of the block kernels (cfg3 block kernel, 1 / 2 / 4: 10.94 / 10.57 / 10.63 ms; smaller CTAs free their slots sooner, 1-warp CTAs hit the 32-CTA limit)

// status bits (device flag word)
constexpr uint32_t ST_BADCODE = 1u;
constexpr uint32_t ST_BADWEIGHT = 2u;
constexpr uint32_t ST_CYCLE = 4u;
constexpr uint32_t ST_BADALPHA = 8u;  // absorption: an alpha of a data cell outside [0,1]
constexpr uint32_t ST_RETRY = 16u;    // the device graph solver ran out of scratch: rerun host-driven

// node flags (per block-exit node)
constexpr uint8_t NF_OUT_TILE = 1;  // target outside the node's tile (FlowExternal at tile level, D22)
constexpr uint8_t NF_DEAD = 2;      // target off-grid or NoData: flow dropped (D8)

// direction code k -> (dx, dy), S:L33 / D1.  Index 0 unused.  Packed 2-bit
// tables (value + 1) so a run-time code costs a shift and a mask.
constexpr uint32_t kDxTab = (1u << 2) | (2u << 4) | (2u << 6) | (2u << 8) | (1u << 10) | (0u << 12) |
                            (0u << 14) | (0u << 16);
constexpr uint32_t kDyTab = (0u << 2) | (0u << 4) | (1u << 6) | (2u << 8) | (2u << 10) | (2u << 12) |
                            (1u << 14) | (0u << 16);
__host__ __device__ constexpr int dir_dx(int k) { return (int)((kDxTab >> (2 * k)) & 3u) - 1; }
__host__ __device__ constexpr int dir_dy(int k) { return (int)((kDyTab >> (2 * k)) & 3u) - 1; }
static_assert(dir_dx(1) == 0 && dir_dy(1) == -1 && dir_dx(2) == 1 && dir_dy(2) == -1 && dir_dx(3) == 1 &&
                  dir_dy(3) == 0 && dir_dx(4) == 1 && dir_dy(4) == 1 && dir_dx(5) == 0 && dir_dy(5) == 1 &&
                  dir_dx(6) == -1 && dir_dy(6) == 1 && dir_dx(7) == -1 && dir_dy(7) == 0 &&
                  dir_dx(8) == -1 && dir_dy(8) == -1,
              "direction table (S:L33)");
// code pointing back: opp(k) = ((k + 3) & 7) + 1
__host__ __device__ constexpr int dir_opp(int k) { return ((k + 3) & 7) + 1; }

// ---------------------------------------------------------------- geometry
// Raster H x W, cut into tiles TH x TW (ragged last row/col, D20), each tile
// cut into blocks BR x BC (ragged at the tile's far edges).  Global block grid
// NBR x NBC = (TR * nbt_r) x (TC * nbt_c); blocks past a ragged tile edge are
// empty (h or w <= 0) and skipped.
struct Geom {
  int64_t H, W;      // raster (or strip) size
  int64_t TH, TW;    // tile size
  int64_t TR, TC;    // tiles
  int64_t nbt_r, nbt_c;  // blocks per tile (rows / cols)
  int64_t NBR, NBC;  // global block grid
  int64_t nblocks;
  int64_t row0;      // global row of this raster's first row (strips)
  int64_t GH;        // global raster rows (== H single GPU)
  int br, bc, pb;    // block shape and perimeter slots per block (2(br+bc)-4)
  int nw;            // warps per block kernel CTA
  int regular;       // blocks tile the tiles exactly (TH % br == 0, TW % bc == 0): a plain block grid

  // Block / tile arithmetic in 32 bits (rows, columns, block ids < 2^32 per
  // device); 64-bit integer division is a long instruction sequence on GPUs.
  __host__ __device__ int64_t tile_of_block(int64_t b) const {
    const uint32_t gr = (uint32_t)b / (uint32_t)NBC, gc = (uint32_t)b % (uint32_t)NBC;
    return (int64_t)(gr / (uint32_t)nbt_r) * TC + gc / (uint32_t)nbt_c;
  }
  // block extent
  __host__ __device__ void block_box(int64_t b, int64_t& y0, int64_t& x0, int& h, int& w) const {
    const uint32_t gr = (uint32_t)b / (uint32_t)NBC, gc = (uint32_t)b % (uint32_t)NBC;
    const uint32_t ty = gr / (uint32_t)nbt_r, tx = gc / (uint32_t)nbt_c;
    y0 = (int64_t)ty * TH + (int64_t)(gr - ty * (uint32_t)nbt_r) * br;
    x0 = (int64_t)tx * TW + (int64_t)(gc - tx * (uint32_t)nbt_c) * bc;
    const int64_t ty1 = ((int64_t)ty + 1) * TH < H ? ((int64_t)ty + 1) * TH : H;
    const int64_t tx1 = ((int64_t)tx + 1) * TW < W ? ((int64_t)tx + 1) * TW : W;
    const int64_t hh = ty1 - y0, ww = tx1 - x0;
    h = hh <= 0 ? 0 : (hh > br ? br : (int)hh);
    w = ww <= 0 ? 0 : (ww > bc ? bc : (int)ww);
  }
  __host__ __device__ int64_t block_of(int64_t y, int64_t x, int& ly, int& lx) const {
    const uint32_t ty = (uint32_t)y / (uint32_t)TH, tx = (uint32_t)x / (uint32_t)TW;
    const uint32_t ry = (uint32_t)y - ty * (uint32_t)TH, rx = (uint32_t)x - tx * (uint32_t)TW;
    const uint32_t qy = ry / (uint32_t)br, qx = rx / (uint32_t)bc;
    ly = (int)(ry - qy * (uint32_t)br);
    lx = (int)(rx - qx * (uint32_t)bc);
    return (int64_t)(ty * (uint32_t)nbt_r + qy) * NBC + tx * (uint32_t)nbt_c + qx;
  }
  __host__ __device__ void tile_box(int64_t t, int64_t& y0, int64_t& x0, int64_t& h,
                                    int64_t& w) const {
    const int64_t ty = (uint32_t)t / (uint32_t)TC, tx = (uint32_t)t % (uint32_t)TC;
    y0 = ty * TH;
    x0 = tx * TW;
    h = (y0 + TH <= H) ? TH : H - y0;
    w = (x0 + TW <= W) ? TW : W - x0;
  }
};

Geom make_geom(int64_t H, int64_t W, int64_t th, int64_t tw, int br);

// ---------------------------------------------------------------- perimeter order
// Clockwise from the top-left: top row L->R, right column, bottom row R->L,
// left column bottom->top; 1-wide boxes are row-major (S:L60-67 convention).
__host__ __device__ inline int64_t perim_count(int64_t h, int64_t w) {
  if (h <= 0 || w <= 0) return 0;
  if (h == 1 || w == 1) return h * w;
  return 2 * (h + w) - 4;
}
__host__ __device__ inline void perim_xy(int64_t p, int64_t h, int64_t w, int64_t& x, int64_t& y) {
  if (h == 1 || w == 1) {
    y = p / w;
    x = p % w;
    return;
  }
  if (p < w) { x = p; y = 0; return; }
  p -= w;
  if (p < h - 1) { x = w - 1; y = p + 1; return; }
  p -= h - 1;
  if (p < w - 1) { x = w - 2 - p; y = h - 1; return; }
  p -= w - 1;
  x = 0;
  y = h - 2 - p;
}
__host__ __device__ inline int64_t perim_index(int64_t x, int64_t y, int64_t h, int64_t w) {
  if (h == 1 || w == 1) return y * w + x;
  if (y == 0) return x;
  if (x == w - 1) return w + y - 1;
  if (y == h - 1) return w + (h - 1) + (w - 2 - x);
  if (x == 0) return w + (h - 1) + (w - 1) + (h - 2 - y);
  return -1;
}

// ---------------------------------------------------------------- D8 (H1)
// Steepest strictly-downhill data neighbour; drops fl32(zc - zn) (D5);
// cardinal vs diagonal by the exact compare 2a^2 > b^2 in fp64 (D4);
// ties to the lowest code (D2); no downhill data neighbour -> lowest
// off-grid/NoData code (outlet, D3), else NoFlow (D6).  `zs` holds staged
// elevations where NoData and off-grid are NaN.
template <int STRIDE>
__device__ __forceinline__ uint8_t d8_code(const float* zs, int i) {
  const float zc = zs[i];
  if (isnan(zc)) return kNoData;
  // drops; a NaN neighbour (NoData / off-grid) gives a NaN drop, which no
  // comparison below accepts, so the common path needs no NaN tests
  float d[9];
#pragma unroll
  for (int k = 1; k <= 8; ++k) d[k] = __fsub_rn(zc, zs[i + dir_dy(k) * STRIDE + dir_dx(k)]);
  // best cardinal / diagonal: strictly larger replaces, so the first
  // (lowest) code wins ties (D2)
  float a = 0.0f, b = 0.0f;
  int kc = 0, kd = 0;
#pragma unroll
  for (int k = 1; k <= 7; k += 2)
    if (d[k] > a) { a = d[k]; kc = k; }
#pragma unroll
  for (int k = 2; k <= 8; k += 2)
    if (d[k] > b) { b = d[k]; kd = k; }
  if (kc && kd) {
    const double da = (double)a, db = (double)b;
    return (uint8_t)(__dmul_rn(__dmul_rn(2.0, da), da) > __dmul_rn(db, db) ? kc : kd);
  }
  if (kc | kd) return (uint8_t)(kc | kd);
  // no downhill data neighbour: outlet through the lowest off-grid / NoData
  // code (D3), else NoFlow (D6)
#pragma unroll
  for (int k = 1; k <= 8; ++k)
    if (isnan(zs[i + dir_dy(k) * STRIDE + dir_dx(k)])) return (uint8_t)k;
  return kNoFlow;
}

__device__ __forceinline__ float stage_z(float v, float nodata) {
  // v*0 + v is v for finite v and NaN for +-inf and NaN (one FMA-pipe op
  // instead of a compare and a select on the ALU pipe, which bounds k_d8v)
  const float f = __fmaf_rn(v, 0.0f, v);
  return v != nodata ? f : __int_as_float(0x7fc00000);
}

// ---------------------------------------------------------------- accumulator traits
template <class T> struct AccT;
template <> struct AccT<uint32_t> {
  __host__ __device__ static uint32_t marker() { return 0xFFFFFFFFu; }
};
template <> struct AccT<unsigned long long> {
  __host__ __device__ static unsigned long long marker() { return ~0ull; }
};
template <> struct AccT<double> {
  __device__ static double marker() { return __longlong_as_double(0x7ff8000000000000ll); }
};

__device__ __forceinline__ void atomic_add(uint32_t* p, uint32_t v) { atomicAdd(p, v); }
__device__ __forceinline__ void atomic_add(unsigned long long* p, unsigned long long v) { atomicAdd(p, v); }
__device__ __forceinline__ void atomic_add(double* p, double v) { atomicAdd(p, v); }

// arguments of the block kernels (pass 1 / pass 2, block.cu)
template <class T, int WK>
struct PassArgs {
  Geom g;
  const float* dem;       // pass 1 from DEM
  float nodata;
  const uint8_t* dirs_in; // pass 1 from dirs, and pass 2
  uint8_t* dirs_out;      // pass 1 from DEM: D8 output (may be null)
  const void* w;          // weights (WK: 0 none, 1 u32, 2 f32)
  // halo rows of a row strip (H7): global rows row0-1 and row0+H, or null
  // when the strip touches the raster edge (then those rows are off-grid)
  const float* dem_up;
  const float* dem_dn;
  const uint8_t* dirs_up;
  const uint8_t* dirs_dn;
  // pass 1 outputs
  uint32_t* node_count;
  T* node_val;
  uint32_t* node_slot;
  uint32_t* node_tgt;
  uint8_t* node_flags;
  uint32_t* slot_root;
  unsigned long long* wsum;
  // pass 2 inputs / outputs
  T* x_slot;              // offsets per block slot (pass 1 adds leaf exits into it; pass 2 reads it)
  T* acc;
  uint32_t* status;
  bool retain;  // pass 1 writes the block-local accumulation into acc (RETAIN)
  bool vsmem;   // block values on chip (k_pass1v / k_pass2v) instead of in acc (FA_OPT_VALUES)
  int64_t b_begin, b_end;  // the launch covers blocks [b_begin, b_end) (chunked: host-buffer pipelining)
  bool cut;     // tile records wanted: slot roots also for every slot on a tile edge
  // absorption: per-cell fraction of A passed on
  // (row-major like acc), the product of alpha along each entry slot's
  // in-block path before its exit, and alpha at each node's exit cell
  const float* alpha;
  T* slot_f;
  float* node_alpha;
};

// warp-aggregated append of `v` (if pred) to list[*count]
__device__ __forceinline__ void warp_append(bool pred, uint32_t v, uint32_t* list, uint32_t* count) {
  const unsigned mask = __ballot_sync(0xFFFFFFFFu, pred);
  if (!mask) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(mask) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(count, (uint32_t)__popc(mask));
  base = __shfl_sync(0xFFFFFFFFu, base, leader);
  if (pred) list[base + __popc(mask & ((1u << lane) - 1))] = v;
}

}  // namespace fa
