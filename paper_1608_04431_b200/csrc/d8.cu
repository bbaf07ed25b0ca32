// d8.cu -- H1 as standalone kernels: the D8 code of every cell of a raster
// (or of a strip plus its halo rows), written as u8 codes for the block
// kernel.  D8 rule: P:L47-48 ("the steepest downslope neighbour"), with the
// readings D2-D6 of DESIGN.md.
#include <cstdlib>

#include "d8.cuh"

namespace fa {

// ---------------------------------------------------------------- standalone D8
// H1 as its own kernel (fa_flowdirs, and the first step of the single-device
// path): a CTA stages a 32 x 128 tile of z with a 1-cell halo (float4 rows),
// then each thread runs the same d8_window down one column with a rolling
// 3x3 register window.  No large shared state, so many warps per SM hide the
// latency of the compare chains.  Rows -1 / H come from dem_up / dem_dn (a
// strip's halo rows) or are off-grid.
constexpr int DR = 32, DC = 128, DZS = DC + 8;  // tile rows / cols, staged row stride (interior at col 4)
__global__ void __launch_bounds__(DC) k_d8(const float* __restrict__ dem, const float* __restrict__ dem_up,
                                           const float* __restrict__ dem_dn, int64_t H, int64_t W, float nodata,
                                           uint8_t* __restrict__ dirs) {
  __shared__ __align__(16) float zs[(DR + 2) * DZS];
  const int64_t y0 = (int64_t)blockIdx.y * DR, x0 = (int64_t)blockIdx.x * DC;
  const int tid = threadIdx.x;
  const float qnan = __int_as_float(0x7fc00000);
  const bool vec = x0 + DC <= W && ((W & 3) == 0) && ((reinterpret_cast<uintptr_t>(dem) & 15) == 0) &&
                   (!dem_up || (reinterpret_cast<uintptr_t>(dem_up) & 15) == 0) &&
                   (!dem_dn || (reinterpret_cast<uintptr_t>(dem_dn) & 15) == 0);
  if (vec) {
    // per row: 32 float4 + 2 halo scalars
    for (int i = tid; i < (DR + 2) * (DC / 4 + 2); i += DC) {
      const int r = i / (DC / 4 + 2), k = i - r * (DC / 4 + 2);
      const float* row = dem_row(dem, dem_up, dem_dn, H, W, y0 + r - 1);
      if (k < DC / 4) {
        float4 v = make_float4(qnan, qnan, qnan, qnan);
        if (row) {
          v = __ldg(reinterpret_cast<const float4*>(row + x0) + k);
          v.x = stage_z(v.x, nodata);
          v.y = stage_z(v.y, nodata);
          v.z = stage_z(v.z, nodata);
          v.w = stage_z(v.w, nodata);
        }
        *reinterpret_cast<float4*>(&zs[r * DZS + 4 + 4 * k]) = v;
      } else {
        const int lx = k == DC / 4 ? -1 : DC;
        const int64_t gx = x0 + lx;
        float v = qnan;
        if (row && gx >= 0 && gx < W) v = stage_z(__ldg(row + gx), nodata);
        zs[r * DZS + 4 + lx] = v;
      }
    }
  } else {
    for (int i = tid; i < (DR + 2) * (DC + 2); i += DC) {
      const int r = i / (DC + 2), lx = i - r * (DC + 2) - 1;
      const float* row = dem_row(dem, dem_up, dem_dn, H, W, y0 + r - 1);
      const int64_t gx = x0 + lx;
      float v = qnan;
      if (row && gx >= 0 && gx < W) v = stage_z(__ldg(row + gx), nodata);
      zs[r * DZS + 4 + lx] = v;
    }
  }
  __syncthreads();
  const int64_t gx = x0 + tid;
  if (gx >= W) return;
  const int rows = (int)(H - y0 < DR ? H - y0 : DR);
  int zi = 4 + tid;
  float u0 = zs[zi - 1], u1 = zs[zi], u2 = zs[zi + 1];
  zi += DZS;
  float c0 = zs[zi - 1], c1 = zs[zi], c2 = zs[zi + 1];
  uint8_t* out = dirs + y0 * W + gx;
#pragma unroll 4
  for (int ly = 0; ly < rows; ++ly) {
    zi += DZS;
    const float e0 = zs[zi - 1], e1 = zs[zi], e2 = zs[zi + 1];
    const int d = d8_window(c1, u1, u2, c2, e2, e1, e0, c0, u0);
    out[ly * W] = (uint8_t)(d == kNoData ? kNoData : (d & 15));
    u0 = c0; u1 = c1; u2 = c2;
    c0 = e0; c1 = e1; c2 = e2;
  }
}

// D8 from precomputed drops (same rule as d8_window): centre NaN -> NoData;
// a NaN drop means a NaN (NoData / off-grid) neighbour.  The best cardinal
// and diagonal drops are maxima (fmaxf ignores NaN), their codes the first
// equal drop in code order (lowest code on ties, D2); strictly downhill
// means > 0; then the exact fp64 compare 2a^2 > b^2 (D4).
__device__ __forceinline__ uint32_t d8_drops(bool cnan, float d1, float d2, float d3, float d4, float d5, float d6,
                                             float d7, float d8) {
  const float a = fmaxf(fmaxf(d1, d3), fmaxf(d5, d7));
  const float b = fmaxf(fmaxf(d2, d4), fmaxf(d6, d8));
  const bool vc = a > 0.0f, vd = b > 0.0f;
  uint32_t code;
  if (vc | vd) {
    bool card = vc;
    if (vc && vd) {
      const double da = (double)a, db = (double)b;
      card = __dmul_rn(__dmul_rn(2.0, da), da) > __dmul_rn(db, db);
    }
    // only the winning group's code is searched: its first drop equal to the
    // group maximum (selects instead of a second compare chain; the ALU pipe
    // bounds this kernel)
    const float m = card ? a : b;
    const float e1 = card ? d1 : d2, e3 = card ? d3 : d4, e5 = card ? d5 : d6;
    uint32_t c = e5 == m ? 5u : 7u;
    c = e3 == m ? 3u : c;
    c = e1 == m ? 1u : c;
    code = c + (card ? 0u : 1u);
  } else {
    // no downhill data neighbour: the lowest NaN neighbour (outlet, D3), else
    // NoFlow.  A NoData centre (all drops NaN) always lands here, so its
    // check costs nothing on the common path.
    code = isnan(d1) ? 1u : isnan(d2) ? 2u : isnan(d3) ? 3u : isnan(d4) ? 4u : isnan(d5) ? 5u
         : isnan(d6) ? 6u : isnan(d7) ? 7u : isnan(d8) ? 8u : (uint32_t)kNoFlow;
    if (cnan) code = kNoData;
  }
  return code;
}

// H1, vectorised: each lane owns 4 adjacent columns of a 128-column warp
// strip and runs down RS rows.  Rows are read as one float4 per lane (the
// two outer columns come from the neighbour lanes by shuffles, or from the
// halo at the warp's edges), and every pairwise drop is computed once:
// fl(z_a - z_b) = -fl(z_b - z_a) exactly under round-to-nearest, so the drop
// to the N / NW / NE neighbour is the negated S / SE / SW drop of the row
// above, and W is the negated E drop of the left cell (D5 unchanged).
constexpr int DV_RS = 32;  // rows per warp
__global__ void __launch_bounds__(128) k_d8v(const float* __restrict__ dem, const float* __restrict__ dem_up,
                                             const float* __restrict__ dem_dn, int64_t H, int64_t W, float nodata,
                                             uint8_t* __restrict__ dirs) {
  const int lane = threadIdx.x & 31;
  const int64_t x0 = ((int64_t)blockIdx.x * 4 + (threadIdx.x >> 5)) * 128;
  if (x0 >= W) return;
  const int64_t y0 = (int64_t)blockIdx.y * DV_RS;
  const int64_t gx = x0 + 4 * lane;
  const bool own = gx < W;
  const float qnan = __int_as_float(0x7fc00000);
  // a row in flight: raw float4 of the lane's columns + the two warp-edge halo values
  // one halo value per row: lane 0 reads the column left of the strip, lane
  // 31 the column right of it (staged once, for both)
  struct Raw {
    float4 v;
    float h;
  };
  const bool hl_ok = lane == 0 && x0 > 0, hr_ok = lane == 31 && x0 + 128 < W;
  const int64_t hx = lane == 0 ? x0 - 1 : x0 + 128;
  auto issue = [&](int64_t gy) {
    Raw q{make_float4(qnan, qnan, qnan, qnan), qnan};
    const float* row = dem_row(dem, dem_up, dem_dn, H, W, gy);
    if (row) {
      if (own) q.v = __ldg(reinterpret_cast<const float4*>(row + gx));
      if (hl_ok || hr_ok) q.h = __ldg(row + hx);
    }
    return q;
  };
  auto finish = [&](const Raw& q, float (&R)[6]) {
    // NoData / non-finite -> NaN (off-grid values are NaN already)
    const float4 v = make_float4(stage_z(q.v.x, nodata), stage_z(q.v.y, nodata), stage_z(q.v.z, nodata),
                                 stage_z(q.v.w, nodata));
    const float hz = stage_z(q.h, nodata);
    const float l = __shfl_up_sync(kFull, v.w, 1), r = __shfl_down_sync(kFull, v.x, 1);
    R[0] = lane == 0 ? hz : l;
    R[1] = v.x;
    R[2] = v.y;
    R[3] = v.z;
    R[4] = v.w;
    R[5] = lane == 31 ? hz : r;
  };
  float P[6], C[6], D[6];
  {
    const Raw q0 = issue(y0 - 1), q1 = issue(y0);
    finish(q0, P);
    finish(q1, C);
  }
  Raw nxt = issue(y0 + 1);  // one row ahead of its use
  // drops between the row above and the current row
  float pv[6], ps[6], pt[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) pv[j] = ps[j] = pt[j] = 0.0f;
#pragma unroll
  for (int j = 1; j <= 4; ++j) pv[j] = __fsub_rn(P[j], C[j]);
#pragma unroll
  for (int j = 0; j <= 4; ++j) ps[j] = __fsub_rn(P[j], C[j + 1]);
#pragma unroll
  for (int j = 1; j <= 5; ++j) pt[j] = __fsub_rn(P[j], C[j - 1]);
  const int rows = (int)(H - y0 < DV_RS ? H - y0 : DV_RS);
  uint8_t* out = dirs + y0 * W + gx;
  for (int r = 0; r < rows; ++r) {
    const Raw cur = nxt;
    nxt = issue(y0 + r + 2);
    finish(cur, D);
    float v[6], sd[6], t[6], hh[6];
#pragma unroll
    for (int j = 0; j < 6; ++j) v[j] = sd[j] = t[j] = hh[j] = 0.0f;
#pragma unroll
    for (int j = 1; j <= 4; ++j) v[j] = __fsub_rn(C[j], D[j]);
#pragma unroll
    for (int j = 0; j <= 4; ++j) sd[j] = __fsub_rn(C[j], D[j + 1]);
#pragma unroll
    for (int j = 1; j <= 5; ++j) t[j] = __fsub_rn(C[j], D[j - 1]);
#pragma unroll
    for (int j = 0; j <= 4; ++j) hh[j] = __fsub_rn(C[j], C[j + 1]);
    uint32_t packed = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j = i + 1;
      // N, NE, E, SE, S, SW, W, NW
      const uint32_t code = d8_drops(isnan(C[j]), -pv[j], -pt[j + 1], hh[j], sd[j], v[j], t[j], -hh[j - 1],
                                     -ps[j - 1]);
      packed += code * (1u << (8 * i));  // an FMA-pipe multiply-add, not ALU shifts/ors
    }
    if (own) *reinterpret_cast<uint32_t*>(out + (int64_t)r * W) = packed;
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      pv[j] = v[j];
      ps[j] = sd[j];
      pt[j] = t[j];
      C[j] = D[j];
    }
  }
}

cudaError_t launch_d8(const float* dem, const float* dem_up, const float* dem_dn, int64_t H, int64_t W,
                      float nodata, uint8_t* dirs, cudaStream_t st) {
  const bool vec = (W % 4) == 0 && ((reinterpret_cast<uintptr_t>(dem) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(dirs) & 3) == 0) &&
                   (!dem_up || (reinterpret_cast<uintptr_t>(dem_up) & 15) == 0) &&
                   (!dem_dn || (reinterpret_cast<uintptr_t>(dem_dn) & 15) == 0);
  if (vec) {
    dim3 grid((unsigned)((W + 511) / 512), (unsigned)((H + DV_RS - 1) / DV_RS));
    k_d8v<<<grid, 128, 0, st>>>(dem, dem_up, dem_dn, H, W, nodata, dirs);
  } else {
    dim3 grid((unsigned)((W + DC - 1) / DC), (unsigned)((H + DR - 1) / DR));
    k_d8<<<grid, DC, 0, st>>>(dem, dem_up, dem_dn, H, W, nodata, dirs);
  }
  return cudaGetLastError();
}

}  // namespace fa
