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
// relaxation from W = +inf: a CTA owns a 32x32 tile, stages W with a 1-cell
// halo in shared memory and runs Gauss-Seidel sweeps until the tile is
// stable; tiles exchange through global memory between launches, each
// launch works through a list of the tiles next to a border that fell in the
// previous one, and the host repeats launches until the list is empty.  NoData (z == nodata or
// non-finite) is copied unchanged and never relaxed.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdint>

#include "fa_internal.cuh"
#include "forest.cuh"

// warps per CTA (rows of threads) for 32x32 and 64x64 tiles
// rows of a thread: consecutive (1, sweeps alternate down / up) or strided
// by TY (0)
#ifndef FA_FILL_CONTIG
#define FA_FILL_CONTIG 1
#endif
#if FA_FILL_CONTIG
#define FILL_ROW(i) (ty * CY + (i))
#else
#define FILL_ROW(i) (ty + TY * (i))
#endif
#ifndef FA_FILL_TY32
#define FA_FILL_TY32 4
#endif
#ifndef FA_FILL_TY64
#define FA_FILL_TY64 16
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

// one launch over a worklist of tiles (a persistent grid strides over
// list_in): each listed tile relaxes to its local fixed point given the
// halo values it stages (a neighbour may already have lowered them this
// launch: any staged value is an upper bound of the fixed point, so the
// relaxation stays monotone).  A tile is at its local fixed point for the
// halo it saw, so it is listed again only when a neighbour lowers a border
// cell facing it: a tile whose border cells fall appends the neighbours on
// those sides to list_out (a corner neighbour needs both of its sides, a
// conservative test), deduplicated by stamping them with the next launch's
// epoch.  A CTA of 32 x TY threads owns an FT x FT tile (FT/TY consecutive
// rows and FT/32 columns of cells per thread).
template <int FT, int TY>
__global__ void __launch_bounds__(32 * TY) k_fill_relax(const float* __restrict__ z, int64_t H, int64_t W,
                                                     float nodata, float* Wg, int nbx, int nby,
                                                     const uint32_t* __restrict__ list_in,
                                                     const uint32_t* __restrict__ cnt_in, uint32_t* list_out,
                                                     uint32_t* cnt_out, uint32_t* stamp, uint32_t epoch) {
  constexpr int CY = FT / TY, CX = FT / 32;
  __shared__ float s[FT + 2][FT + 3];
  __shared__ float zs[FT][FT + 1];  // the tile's elevations (staged once)
  __shared__ uint32_t sides;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const uint32_t ntile = *cnt_in;
  for (uint32_t idx = blockIdx.x; idx < ntile; idx += gridDim.x) {
    const uint32_t tile = list_in[idx];
    const int by = (int)(tile / (uint32_t)nbx), bx = (int)(tile - (uint32_t)by * (uint32_t)nbx);
    const int64_t x0 = (int64_t)bx * FT, y0 = (int64_t)by * FT;
    __syncthreads();  // the previous tile's shared reads are done
    if (threadIdx.x == 0) sides = 0u;
    // stage W (NoData and off-grid act as +inf: never a minimising neighbour)
    for (int i = threadIdx.x; i < (FT + 2) * (FT + 2); i += blockDim.x) {
      const int ly = i / (FT + 2) - 1, lx = i % (FT + 2) - 1;
      const int64_t gy = y0 + ly, gx = x0 + lx;
      float v = INFINITY, zz = INFINITY;
      if (gy >= 0 && gx >= 0 && gy < H && gx < W) {
        zz = z[gy * W + gx];
        const float w = Wg[gy * W + gx];  // both loads in flight together
        if (!f_nodata(zz, nodata)) v = w;
      }
      s[ly + 1][lx + 1] = v;
      if (ly >= 0 && lx >= 0 && ly < FT && lx < FT) zs[ly][lx] = zz;
    }
    __syncthreads();
    float zc[CY][CX], cur[CY][CX], init[CY][CX];
    bool active[CY][CX];
#pragma unroll
    for (int i = 0; i < CY; ++i)
#pragma unroll
      for (int j = 0; j < CX; ++j) {
        const int ly = FILL_ROW(i), lx = tx + 32 * j;
        const float zz = zs[ly][lx];  // +inf off the grid
        active[i][j] = !f_nodata(zz, nodata);  // seeds hold z, their fixed value: relaxing them is a no-op
        zc[i][j] = active[i][j] ? zz : 0.0f;
        cur[i][j] = init[i][j] = active[i][j] ? s[ly + 1][lx + 1] : INFINITY;
      }
    bool any = false;
    for (int it = 0; it < FT * FT; ++it) {
      // Gauss-Seidel: a value is written as soon as it falls; a thread owns
      // CY consecutive rows and walks them down on even sweeps and up on
      // odd ones, so one sweep carries a value across all of them
      bool ch = false;
      auto relax = [&](const int i, const int j) {
        if (active[i][j]) {
          const int ly = FILL_ROW(i), lx = tx + 32 * j;
          float m = INFINITY;
#pragma unroll
          for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int dx = 0; dx < 3; ++dx)
              if (dy != 1 || dx != 1) m = fminf(m, s[ly + dy][lx + dx]);
          const float c = fmaxf(zc[i][j], nextafterf(m, INFINITY));
          if (c < cur[i][j]) {
            cur[i][j] = c;
            s[ly + 1][lx + 1] = c;
            ch = true;
          }
        }
      };
      if (FA_FILL_CONTIG && (it & 1)) {
#pragma unroll
        for (int i = CY - 1; i >= 0; --i)
#pragma unroll
          for (int j = 0; j < CX; ++j) relax(i, j);
      } else {
#pragma unroll
        for (int i = 0; i < CY; ++i)
#pragma unroll
          for (int j = 0; j < CX; ++j) relax(i, j);
      }
      if (!__syncthreads_or(ch)) break;
      any = true;
    }
    if (!any) continue;  // block-uniform
    uint32_t mine = 0u;
#pragma unroll
    for (int i = 0; i < CY; ++i)
#pragma unroll
      for (int j = 0; j < CX; ++j)
        if (active[i][j] && cur[i][j] != init[i][j]) {
          const int ly = FILL_ROW(i), lx = tx + 32 * j;
          Wg[(y0 + ly) * W + x0 + lx] = cur[i][j];
          mine |= (ly == 0 ? 1u : 0u) | (ly == FT - 1 ? 2u : 0u) | (lx == 0 ? 4u : 0u) | (lx == FT - 1 ? 8u : 0u);
        }
    if (mine) atomicOr(&sides, mine);
    __syncthreads();
    if (threadIdx.x < 9 && threadIdx.x != 4) {
      // sides: 1 top, 2 bottom, 4 left, 8 right
      const int dy = (int)threadIdx.x / 3 - 1, dx = (int)threadIdx.x % 3 - 1;
      const uint32_t need = (dy < 0 ? 1u : dy > 0 ? 2u : 0u) | (dx < 0 ? 4u : dx > 0 ? 8u : 0u);
      const int yy = by + dy, xx = bx + dx;
      if ((sides & need) == need && yy >= 0 && xx >= 0 && yy < nby && xx < nbx) {
        const uint32_t nt = (uint32_t)yy * (uint32_t)nbx + (uint32_t)xx;
        if (atomicExch(&stamp[nt], epoch) != epoch) list_out[atomicAdd(cnt_out, 1u)] = nt;
      }
    }
  }
}

__global__ void k_fill_iota(uint32_t* list, uint32_t* cnt, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) list[i] = i;
  if (blockIdx.x == 0 && threadIdx.x == 0) *cnt = n;
}

}  // namespace

// fill z into out (device buffers)
cudaError_t fill_depressions(Runtime& rt, const float* z, int64_t H, int64_t W, float nodata, float* out,
                             int tile) {
  cudaStream_t st = rt.st;
  const int64_t n = H * W;
  k_fill_init<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 64), 256, 0, st>>>(z, H, W, nodata, out);
  ++rt.launches;
  const int FT = tile == 64 ? 64 : 32;  // FA_OPT_FILL_TILE: 32 (default) or 64
  const int nbx = (int)((W + FT - 1) / FT), nby = (int)((H + FT - 1) / FT);
  const uint32_t nt = (uint32_t)nbx * (uint32_t)nby;
  uint32_t* la = rt.alloc<uint32_t>(nt);
  uint32_t* lb = rt.alloc<uint32_t>(nt);
  uint32_t* stamp = rt.alloc<uint32_t>(nt);
  uint32_t* cnt = rt.alloc<uint32_t>(2);
  if (rt.err) return rt.err;
  cudaMemsetAsync(stamp, 0, sizeof(uint32_t) * nt, st);
  k_fill_iota<<<(unsigned)std::min<uint32_t>((nt + 255) / 256, 148 * 8), 256, 0, st>>>(la, cnt, nt);  // every tile
  ++rt.launches;
  uint32_t *ca = cnt, *cb = cnt + 1;
  // persistent grid: as many CTAs as fit per SM (threads and shared memory)
  const int ty = FT == 32 ? FA_FILL_TY32 : FA_FILL_TY64;
  const int per_sm = std::min(2048 / (32 * ty), (228 * 1024) / (int)(sizeof(float) * (FT + 2) * (FT + 3) + 1024));
  const unsigned grid = 148u * (unsigned)std::min(per_sm, 32);
  uint32_t epoch = 0;
  for (;;) {
    for (int j = 0; j < 4; ++j) {
      cudaMemsetAsync(cb, 0, sizeof(uint32_t), st);
      ++epoch;
      if (FT == 32)
        k_fill_relax<32, FA_FILL_TY32><<<grid, 32 * FA_FILL_TY32, 0, st>>>(z, H, W, nodata, out, nbx, nby, la, ca,
                                                                            lb, cb, stamp, epoch);
      else
        k_fill_relax<64, FA_FILL_TY64><<<grid, 32 * FA_FILL_TY64, 0, st>>>(z, H, W, nodata, out, nbx, nby, la, ca,
                                                                            lb, cb, stamp, epoch);
      std::swap(la, lb);
      std::swap(ca, cb);
    }
    rt.launches += 4;
    rt.read(ca, 1);  // the next launch's worklist size
    if (!rt.h_cnt[0] || rt.err) break;
    // bug catch only: a launch runs only while some value still falls, and a
    // winding depression needs about (path length / tile side) launches, so
    // the bound is the cell count (the old 4(H+W) guard was reachable)
    if ((uint64_t)epoch > (uint64_t)H * (uint64_t)W + 64u) {
      rt.err = cudaErrorUnknown;
      break;
    }
  }
  rt.free(la);
  rt.free(lb);
  rt.free(stamp);
  rt.free(cnt);
  return rt.err ? rt.err : cudaGetLastError();
}

}  // namespace fa
