// d8.cuh -- D8 stencil helpers shared by the fused block kernel (block.cu)
// and the standalone stencil kernels (d8.cu): H1, P:L47-48 + D2-D6.
#pragma once
#include "fa_internal.cuh"

namespace fa {

constexpr unsigned kFull = 0xFFFFFFFFu;

// ---------------------------------------------------------------- H1 core
// D8 of one cell from its 3x3 window (NaN = NoData / off-grid): steepest
// strictly-downhill data neighbour, drops fl32(zc - zn) (D5), cardinal vs
// diagonal by the exact compare 2a^2 > b^2 in fp64 (D4), ties to the lowest
// code (D2); none -> lowest NaN neighbour (outlet, D3; returned | 16: the
// target is NoData), else NoFlow (D6).
__device__ __forceinline__ int d8_window(float zc, float zN, float zNE, float zE, float zSE, float zS,
                                         float zSW, float zW, float zNW) {
  if (isnan(zc)) return kNoData;
  const float d1 = __fsub_rn(zc, zN), d3 = __fsub_rn(zc, zE), d5 = __fsub_rn(zc, zS), d7 = __fsub_rn(zc, zW);
  const float d2 = __fsub_rn(zc, zNE), d4 = __fsub_rn(zc, zSE), d6 = __fsub_rn(zc, zSW),
              d8 = __fsub_rn(zc, zNW);
  // NaN drops fail every comparison; strictly-larger replaces: lowest code wins ties
  float a = 0.0f, b = 0.0f;
  int kc = 0, kd = 0;
  if (d1 > a) { a = d1; kc = 1; }
  if (d3 > a) { a = d3; kc = 3; }
  if (d5 > a) { a = d5; kc = 5; }
  if (d7 > a) { a = d7; kc = 7; }
  if (d2 > b) { b = d2; kd = 2; }
  if (d4 > b) { b = d4; kd = 4; }
  if (d6 > b) { b = d6; kd = 6; }
  if (d8 > b) { b = d8; kd = 8; }
  if (kc && kd) {
    const double da = (double)a, db = (double)b;
    return __dmul_rn(__dmul_rn(2.0, da), da) > __dmul_rn(db, db) ? kc : kd;
  }
  if (kc | kd) return kc | kd;
  int k = kNoFlow;
  if (isnan(zN)) k = 1;
  else if (isnan(zNE)) k = 2;
  else if (isnan(zE)) k = 3;
  else if (isnan(zSE)) k = 4;
  else if (isnan(zS)) k = 5;
  else if (isnan(zSW)) k = 6;
  else if (isnan(zW)) k = 7;
  else if (isnan(zNW)) k = 8;
  return k ? (k | 16) : kNoFlow;
}

// successor word of in-block cell i with code d (| 16: the target is
// NoData); `forb` = direction codes that leave the block from this cell

__device__ __forceinline__ const float* dem_row(const float* dem, const float* up, const float* dn, int64_t H,
                                                int64_t W, int64_t gy) {
  if (gy < -1 || gy > H) return nullptr;
  if (gy == -1) return up;
  if (gy == H) return dn;
  return dem + gy * W;
}

}  // namespace fa
