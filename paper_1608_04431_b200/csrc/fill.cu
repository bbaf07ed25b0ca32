// fill.cu -- depression filling on the GPU ("the
// depressions can be filled to the level of their lowest outlets ...
// Priority-Flood", D15 with the epsilon step nextafterf).
//
// The Priority-Flood+epsilon surface is the unique fixed point
//   W(s) = z(s)                                         seeds s (data cells on
//          the grid edge or 8-adjacent to NoData),
//   W(p) = max(z(p), nextafterf(min_{data n in N8(p)} W(n), +inf))  otherwise,
// (each step strictly raises the cost, so it is a shortest-path fixpoint and
// any schedule converges to the same bits).  The GPU computes it by monotone
// relaxation from W = +inf: a CTA owns a 64x64 tile, stages W with a 1-cell
// halo in shared memory and runs Jacobi sweeps until the tile is stable;
// tiles exchange through global memory between launches, and the host
// repeats launches until no tile changes.  NoData (z == nodata or
// non-finite) is copied unchanged and never relaxed.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdint>

#include "fa_internal.cuh"
#include "forest.cuh"

// Gauss-Seidel sweeps inside a tile (values written as soon as they fall);
// 0 = Jacobi (two-phase, one extra barrier per sweep)
#ifndef FA_FILL_GS
#define FA_FILL_GS 1
#endif

namespace fa {

namespace {


__device__ __forceinline__ bool f_nodata(float v, float nodata) { return !isfinite(v) || v == nodata; }

// W = z at seeds and NoData, +inf elsewhere
__global__ void k_fill_init(const float* __restrict__ z, int64_t H, int64_t W, float nodata, float* out) {
  const int64_t n = H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = z[i];
    if (f_nodata(v, nodata)) {
      out[i] = v;
      continue;
    }
    const int64_t y = i / W, x = i - y * W;
    bool seed = y == 0 || x == 0 || y == H - 1 || x == W - 1;
    for (int dy = -1; dy <= 1 && !seed; ++dy)
      for (int dx = -1; dx <= 1 && !seed; ++dx)
        if ((dy | dx) && f_nodata(z[(y + dy) * W + x + dx], nodata)) seed = true;
    out[i] = seed ? v : INFINITY;
  }
}

// one launch: every tile next to a border that fell in the previous launch
// (dirty_in) relaxes to its local fixed point given the halo values it
// stages (a neighbour may already have lowered them this launch: any staged
// value is an upper bound of the fixed point, so the relaxation stays
// monotone); a tile whose border cells fall records those sides in dirty_out
// and sets *changed.  A CTA of 32x32 threads owns an FT x FT tile
// (C = FT/32 cells per thread and axis): larger tiles carry the fill further
// per launch.
template <int FT>
__global__ void __launch_bounds__(1024) k_fill_relax(const float* __restrict__ z, int64_t H, int64_t W,
                                                     float nodata, float* Wg, uint32_t* changed,
                                                     const uint8_t* __restrict__ dirty_in, uint8_t* dirty_out) {
  constexpr int C = FT / 32;
  __shared__ float s[FT + 2][FT + 3];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t x0 = (int64_t)blockIdx.x * FT, y0 = (int64_t)blockIdx.y * FT;
  {
    // settled neighbourhood: nothing can change here this launch
    const int bx = (int)blockIdx.x, by = (int)blockIdx.y, nbx = (int)gridDim.x, nby = (int)gridDim.y;
    // a tile is at its local fixed point for the halo it last saw: it runs
    // again only if a neighbour changed a border cell facing it (dirty_in
    // holds per tile the sides whose cells fell: 1 top, 2 bottom, 4 left,
    // 8 right; a corner needs both of its sides, a conservative test; 16
    // runs the tile itself, set for the first launch)
    bool dirty = false;
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int yy = by + dy, xx = bx + dx;
        if ((dy | dx) == 0) {
          if (dirty_in[(int64_t)by * nbx + bx] & 16u) dirty = true;  // the first launch
          continue;
        }
        if (yy < 0 || xx < 0 || yy >= nby || xx >= nbx) continue;
        const uint32_t need = (dy < 0 ? 2u : dy > 0 ? 1u : 0u) | (dx < 0 ? 8u : dx > 0 ? 4u : 0u);
        if ((dirty_in[(int64_t)yy * nbx + xx] & need) == need) dirty = true;
      }
    if (!dirty) return;  // block-uniform
  }
  // stage W (NoData and off-grid act as +inf: never a minimising neighbour)
  for (int i = threadIdx.x; i < (FT + 2) * (FT + 2); i += blockDim.x) {
    const int ly = i / (FT + 2) - 1, lx = i % (FT + 2) - 1;
    const int64_t gy = y0 + ly, gx = x0 + lx;
    float v = INFINITY;
    if (gy >= 0 && gx >= 0 && gy < H && gx < W) {
      const float zz = z[gy * W + gx];
      if (!f_nodata(zz, nodata)) v = Wg[gy * W + gx];
    }
    s[ly + 1][lx + 1] = v;
  }
  float zc[C][C], cur[C][C], init[C][C];
  bool active[C][C];
#pragma unroll
  for (int i = 0; i < C; ++i)
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const int ly = ty + 32 * i, lx = tx + 32 * j;
      const int64_t gy = y0 + ly, gx = x0 + lx;
      zc[i][j] = 0.0f;
      cur[i][j] = init[i][j] = INFINITY;
      active[i][j] = false;
      if (gy < H && gx < W) {
        const float zz = z[gy * W + gx];
        if (!f_nodata(zz, nodata)) {
          zc[i][j] = zz;
          cur[i][j] = init[i][j] = Wg[gy * W + gx];
          active[i][j] = true;  // seeds hold z, their fixed value: relaxing them is a no-op
        }
      }
    }
  __syncthreads();
  bool any = false;
  for (int it = 0; it < FT * FT; ++it) {
    float cand[C][C];
    bool ch = false;
#pragma unroll
    for (int i = 0; i < C; ++i)
#pragma unroll
      for (int j = 0; j < C; ++j) {
        cand[i][j] = cur[i][j];
        if (active[i][j]) {
          const int ly = ty + 32 * i, lx = tx + 32 * j;
          float m = INFINITY;
#pragma unroll
          for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int dx = 0; dx < 3; ++dx)
              if (dy != 1 || dx != 1) m = fminf(m, s[ly + dy][lx + dx]);
          const float c = fmaxf(zc[i][j], nextafterf(m, INFINITY));
          if (c < cur[i][j]) {
            cand[i][j] = c;
            ch = true;
#if FA_FILL_GS
            cur[i][j] = c;
            s[ly + 1][lx + 1] = c;
#endif
          }
        }
      }
#if !FA_FILL_GS
    __syncthreads();
    if (ch) {
#pragma unroll
      for (int i = 0; i < C; ++i)
#pragma unroll
        for (int j = 0; j < C; ++j)
          if (cand[i][j] < cur[i][j]) {
            cur[i][j] = cand[i][j];
            s[ty + 32 * i + 1][tx + 32 * j + 1] = cand[i][j];
          }
    }
#endif
    if (!__syncthreads_or(ch)) break;
    any = true;
  }
  if (any) {  // block-uniform
    __shared__ uint32_t sides;
    if (threadIdx.x == 0) sides = 0u;
    __syncthreads();
    uint32_t mine = 0u;
#pragma unroll
    for (int i = 0; i < C; ++i)
#pragma unroll
      for (int j = 0; j < C; ++j)
        if (active[i][j] && cur[i][j] != init[i][j]) {
          const int ly = ty + 32 * i, lx = tx + 32 * j;
          Wg[(y0 + ly) * W + x0 + lx] = cur[i][j];
          mine |= (ly == 0 ? 1u : 0u) | (ly == FT - 1 ? 2u : 0u) | (lx == 0 ? 4u : 0u) | (lx == FT - 1 ? 8u : 0u);
        }
    if (mine) atomicOr(&sides, mine);
    __syncthreads();
    if (threadIdx.x == 0 && sides) {
      atomicOr(changed, 1u);
      dirty_out[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = (uint8_t)sides;
    }
  }
}

}  // namespace

// fill z into out (device buffers)
cudaError_t fill_depressions(Runtime& rt, const float* z, int64_t H, int64_t W, float nodata, float* out) {
  cudaStream_t st = rt.st;
  const int64_t n = H * W;
  k_fill_init<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 64), 256, 0, st>>>(z, H, W, nodata, out);
  ++rt.launches;
  uint32_t* flag = rt.alloc<uint32_t>(1);
  const char* e = getenv("FA_FILL_TILE");  // tuning: 32 or 64 (default)
  const int FT = e && atoi(e) == 32 ? 32 : 64;
  const dim3 grid((unsigned)((W + FT - 1) / FT), (unsigned)((H + FT - 1) / FT));
  const int64_t nt = (int64_t)grid.x * grid.y;
  uint8_t* da = rt.alloc<uint8_t>(nt);
  uint8_t* db = rt.alloc<uint8_t>(nt);
  if (rt.err) return rt.err;
  cudaMemsetAsync(da, 0x1F, nt, st);  // every tile is dirty at the start
  for (int64_t round = 0;; round += 4) {
    cudaMemsetAsync(flag, 0, sizeof(uint32_t), st);
    for (int j = 0; j < 4; ++j) {
      cudaMemsetAsync(db, 0, nt, st);
      if (FT == 32) k_fill_relax<32><<<grid, 1024, 0, st>>>(z, H, W, nodata, out, flag, da, db);
      else k_fill_relax<64><<<grid, 1024, 0, st>>>(z, H, W, nodata, out, flag, da, db);
      std::swap(da, db);
    }
    rt.launches += 4;
    rt.read(flag, 1);
    if (!rt.h_cnt[0] || rt.err) break;
    if (round > 4 * (H + W)) {  // cannot happen: each pass settles at least one more tile ring
      rt.err = cudaErrorUnknown;
      break;
    }
  }
  rt.free(flag);
  rt.free(da);
  rt.free(db);
  return rt.err ? rt.err : cudaGetLastError();
}

}  // namespace fa
