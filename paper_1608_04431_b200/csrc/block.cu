// block.cu -- warp-resident block kernels (SURVEY N1 "SMEM-resident fused tile
// kernel"): each WARP owns one R x 32 block of the raster (R = 16 or 32) and
// runs the paper's single-tile algorithm on it entirely in shared memory,
// with no CTA-wide barrier (only __syncwarp), so blocks never wait on one
// another.
//
//   pass 1 (k_pass1): [H1 D8 from the DEM, 2-cell halo] -> [successor words,
//     H2 in-block donor masks by an 8-neighbour SWAR gather (no atomics),
//     source queue] -> [H3 in-block accumulation, Alg. 1 P:L127-176] ->
//     [H4 block perimeter records: one node per block exit cell with its
//     block-local accumulation, and for the perimeter cells other blocks can
//     drain into, the exit their in-block path reaches (Alg. 2)].
//     RETAIN writes the block-local accumulation to the output here.
//   pass 2 (k_pass2): [H6 offset propagation, EVICT P:L255-262]: rerun H2-H3
//     from the directions with w + x at the block perimeter cells (x =
//     external inbound flow, D11/D12), write A.
//
// By default H1 runs first as its own kernel (d8.cu, k_d8v) and pass 1 reads
// the codes (FROM_DEM = false); FA_FUSED=1 keeps D8 inside pass 1:
//
// Lane layout (fused D8).  Lane l owns column l of the block: the D8 stencil runs down
// the column with a rolling 3x3 register window (3 shared loads per cell
// instead of 9), writing the code and the cell's successor word.  The 2-cell
// halo lets the warp also evaluate D8 on the ring of cells around the block,
// which says which perimeter cells are entries (have a donor outside the
// block): only those need an Alg. 2 walk for the block-exit graph.
//
// Successor word (u16 per cell, block-local index i = 32*ly + lx):
//   bit 15 STOP  -- no in-block successor (NoFlow, NoData, drains into
//                   in-block NoData (D8), or leaves the block);
//   bit 14 EXIT  -- (with STOP) the target is outside the block: a block exit;
//   bits 0-10    -- target index (without STOP).
//
// Values live in the output raster itself: the block's A(p) are accumulated
// in place in acc (global memory; the block's rows stay in L2 while the warp
// works on them), with native global atomics for the pushes.  Shared memory
// holds only the 1-byte codes, successor words, pending counts and the
// queue (~6 KB per warp), so many blocks are in flight per SM to hide the
// L2 latency.  This is RETAIN: acc ends pass 1 holding A_blk.
//
// H3 scheduling: Alg. 1's queue, level-free.  The warp keeps
// one FIFO of ready cells in shared memory, seeded with the sources (cells
// with no in-block donor).  Each iteration every lane pops one ready cell
// (its value is final), adds the value into its successor with an atomic
// and decrements the successor's pending-donor count; the lane that takes
// the count to zero appends the successor (ballot + popc, no queue
// atomics).  One branch-free path per iteration, so all 32 lanes do useful
// work whenever 32 cells are ready.  Visibility: each iteration starts with
// __syncwarp (memory ordering among the warp's lanes, global memory
// included), and a cell appended in one iteration is popped in a later one.
// fp64 sums follow the arrival order; any order is within D13.
#include <cstdlib>

#include "d8.cuh"

namespace fa {

#ifndef FA_FIN_STEPS
#define FA_FIN_STEPS 4  // successor-byte walks: 1 / 4 steps per refill round -> 3.20 / 2.95 ms (cfg3)
#endif
#ifndef FA_FIN_PREFETCH
// L2 prefetches per block row at the start of the finalize (0: none).  cfg3:
// 0 / 1 / 2 / 4 / 8 -> 3.85 / 3.81 / 3.11 / 3.07 / 3.10 ms with the code
// walks; with the successor-byte walks 2 / 4 -> 2.92 / 3.14 ms
#define FA_FIN_PREFETCH 2
#endif
#ifndef FA_FIN_NW
#define FA_FIN_NW 2  // warps (blocks) per CTA of the finalize (4 / 2: cfg3 2.85 / 2.81 ms)
#endif
#ifndef FA_P1_KPW
#define FA_P1_KPW 1  // blocks per warp of pass 1 (interleaved over the launch)
#endif
#ifndef FA_FIN_SMEM_FLOOR
#define FA_FIN_SMEM_FLOOR 6144  // finalize: shared-memory bytes per warp at least (caps the warps per SM)
#endif
#ifndef FA_REC_STEPS
#define FA_REC_STEPS 8  // entry walks: path steps per refill round (4 / 6 / 8 / 16: cfg3 block kernel 10.76 / 10.70 / 10.67 / 10.67 ms)
#endif
#ifndef FA_CHAIN_TAIL
#define FA_CHAIN_TAIL 48  // queue width below which the loop switches to chain bursts (0: never; 32 / 48 with the whole-block kernel: 10.67 / 10.63 ms)
#endif
#ifndef FA_CHAIN_K
#define FA_CHAIN_K 4
#endif
#ifndef FA_P1_MINB
#define FA_P1_MINB 9  // CTAs of 4 warps per SM: 9 (56 registers, 36 warps) vs 8 (64, 32): cfg3 block kernel 12.06 vs 12.21 ms
#endif
#ifndef FA_PEND_BYTES
#define FA_PEND_BYTES 0  // pending counts: 4 bits per cell (0) or a byte (1: cfg3 block kernel 13.38 vs 11.97 ms)
#endif
#ifndef FA_P1_PREFETCH
#define FA_P1_PREFETCH 1  // pass 1 L2 prefetches: 1 the block's weight rows, 2 the neighbours' entry offsets
#endif
constexpr uint8_t kOut = 254;  // ring cell: outside the block, data

// Successor byte of an in-block cell.  A cell that continues to an
// in-block data target holds its code's block offset biased by SB_BIAS
// (31..97, bit 7 clear), so a step is one compare (sb_go) and one add
// (WBT::target).  Stops have bit 7 set: SB_STOP (NoFlow), SB_STOP | SB_DROP
// (drains into in-block NoData: the flow is dropped, D8), SB_STOP | SB_EXIT
// (the code leaves the block: a block exit); NoData cells keep 255.
constexpr uint32_t SB_BIAS = 64u, SB_STOP = 0x80u, SB_DROP = 0x10u, SB_EXIT = 0x20u;
__device__ __forceinline__ bool sb_go(uint32_t sb) { return sb < SB_STOP; }
// a data cell's successor byte says it leaves the block (255 also matches: callers know the cell is data)
__device__ __forceinline__ bool sb_exit(uint32_t sb) { return (sb & (SB_STOP | SB_EXIT)) == (SB_STOP | SB_EXIT); }
// direction codes (bit k) leaving a cell through its N / S / W / E side
constexpr uint32_t DM_N = (1u << 1) | (1u << 2) | (1u << 8);
constexpr uint32_t DM_S = (1u << 4) | (1u << 5) | (1u << 6);
constexpr uint32_t DM_W = (1u << 6) | (1u << 7) | (1u << 8);
constexpr uint32_t DM_E = (1u << 2) | (1u << 3) | (1u << 4);

// packed 8-bit offsets of direction codes 1..8 for a row stride S, plus a
// per-byte bias (0: signed offsets; SB_BIAS: the successor-byte encoding)
__host__ __device__ constexpr uint64_t pack_offsets(int S, int bias = 0) {
  uint64_t t = 0;
  for (int k = 1; k <= 8; ++k)
    t |= (uint64_t)(uint8_t)(int8_t)(dir_dy(k) * S + dir_dx(k) + bias) << (8 * (k - 1));
  return t;
}

template <int R>
struct WBT {
  static constexpr int BR = R, BC = 32, BN = BR * BC;
  static constexpr int PB = 2 * (BR + BC) - 4;
  static constexpr int HS = 36, HOFF = 4;   // dirh: row stride, interior column (4-B aligned rows); the right
                                            // ring cell of a row is byte 0 of the next row
  static constexpr int HN = (BR + 2) * HS + 16;
  static constexpr int ZS = 40, ZOFF = 4;   // z window: row stride, interior column (16-B aligned)
  static constexpr int ZR = BR + 4;         // window rows: 2-cell halo
  static constexpr int ZN = ZR * ZS;
  static constexpr uint64_t OFFH = pack_offsets(HS);
  static constexpr uint64_t OFFA = pack_offsets(BC);
  static constexpr uint64_t OFFB = pack_offsets(BC, (int)SB_BIAS);  // successor bytes of codes 1..8
  static_assert(BC + 1 + SB_BIAS < SB_STOP && SB_BIAS > BC + 1, "biased offsets fit below SB_STOP");
  __device__ static __forceinline__ int offH(int d) { return (int)(int8_t)(OFFH >> (8 * (d - 1))); }
  __device__ static __forceinline__ int offA(int d) { return (int)(int8_t)(OFFA >> (8 * (d - 1))); }
  __device__ static __forceinline__ uint32_t offB(int d) { return (uint32_t)(uint8_t)(OFFB >> (8 * (d - 1))); }
  // in-block target of cell c from its (continuing) successor byte sb
  __device__ static __forceinline__ uint32_t target(uint32_t c, uint32_t sb) { return c + sb - SB_BIAS; }
  __device__ static __forceinline__ int hidx(int ly, int lx) { return (ly + 1) * HS + HOFF + lx; }
  __device__ static __forceinline__ int zidx(int ly, int lx) { return (ly + 2) * ZS + ZOFF + lx; }
  static constexpr int NJ = (PB + 31) / 32;  // perimeter slots per lane
  static constexpr int NP = NJ * 32;         // perimeter slots rounded to whole warps
  static_assert(HS <= 120 && ZS <= 120, "int8 offsets");
  static_assert(PB < 255 && NJ <= 8, "perimeter slots: u8 indices (0xFF = none), at most 8 per lane");
  static_assert(BN <= 2048, "11-bit successor index");
};

template <class T, int R, bool Z>
struct __align__(16) WSmem {
  using WB = WBT<R>;
  using VT = T;
  static constexpr int RR = R;
  static constexpr bool kValues = false;  // values live in global memory (acc), not here
  struct __align__(16) U {
    float z[Z ? WB::ZN : 4];  // z window (fused D8 only)
  } u;
  __device__ __forceinline__ float* zwin() { return u.z; }
  uint8_t dirh[WB::HN];
  uint32_t pend[WB::BN / (FA_PEND_BYTES ? 4 : 8)];  // pending in-block donor counts (<= 8): a byte / 4 bits per cell
  alignas(8) uint8_t sb[WB::BN];  // successor bytes
  // ready queue of Alg. 1 (sources first; each cell enters at most once);
  // after the queue loop: [0,NP) slot -> node id, [NP,2NP) per exit slot:
  // outside donors of the entries draining to it
  alignas(16) uint16_t src[WB::BN];
  alignas(4) uint8_t need[WB::NP];  // per perimeter slot: donors outside the block (ring cells draining in)
#ifdef FA_SMEM_PAD
  uint8_t pad_[FA_SMEM_PAD];  // tuning builds only: extra shared memory per warp
#endif
  __device__ __forceinline__ uint32_t* slot_nid() { return reinterpret_cast<uint32_t*>(src); }
  static_assert(WB::BN * 2 >= 2 * WB::NP * 4, "records scratch lives in the queue");
};

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
// pending in-block donor count of cell t (Alg. 1's D(t)), and its decrement
// (true for the last pending donor: t is ready).  Counts never borrow across
// cells: a count is decremented only while it is >= 1.
__device__ __forceinline__ uint32_t pend_get(const uint32_t* pend, uint32_t t) {
#if FA_PEND_BYTES
  return reinterpret_cast<const uint8_t*>(pend)[t];
#else
  return (pend[t >> 3] >> ((t & 7u) * 4u)) & 0xFu;
#endif
}
__device__ __forceinline__ bool pend_dec(uint32_t* pend, uint32_t t) {
#if FA_PEND_BYTES
  const uint32_t sh = (t & 3u) * 8u;
  const uint32_t old = atomicAdd(&pend[t >> 2], 0u - (1u << sh));
  return ((old >> sh) & 0xFFu) == 1u;
#else
  const uint32_t sh = (t & 7u) * 4u;
  const uint32_t old = atomicAdd(&pend[t >> 3], 0u - (1u << sh));
  return ((old >> sh) & 0xFu) == 1u;
#endif
}
// +1 on byte p of a 4-aligned byte array (counts stay < 256)
__device__ __forceinline__ void need_inc(uint8_t* need, int p) {
  atomicAdd(reinterpret_cast<uint32_t*>(need) + (p >> 2), 1u << (8 * (p & 3)));
}

template <int WK>
__device__ __forceinline__ bool weight_ok(float v) {
  return WK != 2 || (isfinite(v) && v >= 0.0f);  // D21
}

// in-block perimeter order (clockwise from the top-left), ints
__device__ __forceinline__ void bperim_xy(int p, int h, int w, int& x, int& y) {
  if (h == 1 || w == 1) { y = p / w; x = p - y * w; return; }
  if (p < w) { x = p; y = 0; return; }
  p -= w;
  if (p < h - 1) { x = w - 1; y = p + 1; return; }
  p -= h - 1;
  if (p < w - 1) { x = w - 2 - p; y = h - 1; return; }
  p -= w - 1;
  x = 0;
  y = h - 2 - p;
}
__device__ __forceinline__ int bperim_count(int h, int w) {
  if (h <= 0 || w <= 0) return 0;
  if (h == 1 || w == 1) return h * w;
  return 2 * (h + w) - 4;
}
__device__ __forceinline__ int bperim_index(int x, int y, int h, int w) {
  if (h == 1 || w == 1) return y * w + x;
  if (y == 0) return x;
  if (x == w - 1) return w + y - 1;
  if (y == h - 1) return w + (h - 1) + (w - 2 - x);
  return w + (h - 1) + (w - 1) + (h - 2 - y);
}


// successor byte from a D8 result d (| 16: the outlet fallback, the target
// is NoData) and the codes that leave the block from this cell (forb)
__device__ __forceinline__ uint32_t succ_byte(int d, uint32_t forb) {
  const int k = d & 15;
  if (d == kNoData) return kNoData;
  if (k == 0) return SB_STOP;
  if ((forb >> k) & 1u) return SB_STOP | SB_EXIT;
  if (d & 16) return SB_STOP | SB_DROP;  // drains into in-block NoData: dropped (D8)
  return WBT<32>::offB(k);
}

__device__ __forceinline__ uint32_t forb_col(int lx, int w) {
  return (lx == 0 ? DM_W : 0u) | (lx == w - 1 ? DM_E : 0u);
}
__device__ __forceinline__ uint32_t forb_row(int ly, int h) {
  return (ly == 0 ? DM_N : 0u) | (ly == h - 1 ? DM_S : 0u);
}

// byte-permute selectors (code - 1 per nibble) of a word of 4 codes, and
// 0x01 in the bytes whose code leaves a full BR x 32 block (word at row ly,
// columns lx0..lx0+3): a per-byte lookup of the codes leaving through each side
__device__ __forceinline__ uint32_t code_nibbles(uint32_t c1) {
  const uint32_t sel = __vsub4(c1, 0x01010101u) & 0x07070707u;  // code - 1 per byte (no borrow)
  return (sel & 7u) | ((sel >> 4) & 0x70u) | ((sel >> 8) & 0x700u) | ((sel >> 12) & 0x7000u);
}
template <int BR>
__device__ __forceinline__ uint32_t border_exits(uint32_t nib, int ly, int lx0) {
  uint32_t ex4 = 0;
  if (ly == 0) ex4 |= __byte_perm(0x00000101u, 0x01000000u, nib);           // N, NE, NW
  if (ly == BR - 1) ex4 |= __byte_perm(0x01000000u, 0x00000101u, nib);      // SE, S, SW
  if (lx0 == 0) ex4 |= __byte_perm(0u, 0x01010100u, nib) & 0xFFu;           // SW, W, NW (cell 0)
  if (lx0 == 32 - 4) ex4 |= __byte_perm(0x01010100u, 0u, nib) & 0xFF000000u;  // NE, E, SE (cell 3)
  return ex4;
}

// four successor bytes of a full block's word: codes c1 (0..8, NoData 255),
// the byte-permute selectors nib (code - 1 per nibble) and ex4 (0x01 in the
// bytes whose code leaves the block)
__device__ __forceinline__ uint32_t sb_word(uint32_t c1, uint32_t nib, uint32_t ex4) {
  const uint32_t offs = __byte_perm((uint32_t)WBT<32>::OFFB, (uint32_t)(WBT<32>::OFFB >> 32), nib);
  const uint32_t nz = ((((c1 & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | c1) >> 7) & 0x01010101u;  // bytes != 0
  const uint32_t nd = ((c1 >> 7) & 0x01010101u) * 0xFFu;  // NoData bytes (codes are <= 8 otherwise)
  const uint32_t go = ((nz & ~ex4) * 0xFFu) & ~nd;         // continuing cells
  const uint32_t stop = 0x80808080u | ((ex4 & nz) << 5) | nd;  // SB_STOP [| SB_EXIT]; NoData 255
  return (offs & go) | (stop & ~go);
}

// ---------------------------------------------------------------- staging
template <class S>
__device__ __forceinline__ void init_smem(S& s) {
  constexpr int R = S::RR;
  uint32_t* D = reinterpret_cast<uint32_t*>(s.dirh);
  const int lane = lane_id();
  for (int i = lane; i < WBT<R>::HN / 4; i += 32) D[i] = 0xFFFFFFFFu;
  for (int i = lane; i < WBT<R>::NP / 4; i += 32) reinterpret_cast<uint32_t*>(s.need)[i] = 0u;
}


// z window (block + 2-cell halo; NoData / off-grid -> NaN).  Rows of a strip
// halo come from dem_up / dem_dn (H7); rows beyond those read as NaN and the
// ring D8 treats them as unknown (see ring_entries).
template <class T, int WK, class S>
__device__ __forceinline__ void stage_z(S& s, const PassArgs<T, WK>& P, int64_t y0, int64_t x0, int h, int w) {
  using WB = typename S::WB;
  float* zw = s.zwin();
  const Geom& g = P.g;
  const int lane = lane_id();
  const float qnan = __int_as_float(0x7fc00000);
  const bool vec = w == WB::BC && x0 >= 4 && x0 + WB::BC + 4 <= g.W && ((x0 & 3) == 0) && ((g.W & 3) == 0) &&
                   ((reinterpret_cast<uintptr_t>(P.dem) & 15) == 0) &&
                   (!P.dem_up || (reinterpret_cast<uintptr_t>(P.dem_up) & 15) == 0) &&
                   (!P.dem_dn || (reinterpret_cast<uintptr_t>(P.dem_dn) & 15) == 0);
  const int rows = h + 4;
  if (vec) {
    // per window row: 10 float4 covering columns x0-4 .. x0+35; lanes 0..29
    // take 3 rows x 10 quads per round
    const int rr = lane / 10, k = lane - rr * 10;
    if (rr < 3) {
      for (int r = rr; r < rows; r += 3) {
        const float* row = dem_row(P.dem, P.dem_up, P.dem_dn, g.H, g.W, y0 + r - 2);
        float4 v = make_float4(qnan, qnan, qnan, qnan);
        if (row) {
          v = __ldg(reinterpret_cast<const float4*>(row + x0 - 4) + k);
          v.x = fa::stage_z(v.x, P.nodata);
          v.y = fa::stage_z(v.y, P.nodata);
          v.z = fa::stage_z(v.z, P.nodata);
          v.w = fa::stage_z(v.w, P.nodata);
        }
        *reinterpret_cast<float4*>(&zw[r * WB::ZS + 4 * k]) = v;
      }
    }
  } else {
    const int ww = w + 4;
    for (int i = lane; i < rows * ww; i += 32) {
      const int r = i / ww, c = i - r * ww, ly = r - 2, lx = c - 2;
      const int64_t gx = x0 + lx;
      const float* row = dem_row(P.dem, P.dem_up, P.dem_dn, g.H, g.W, y0 + ly);
      float v = qnan;
      if (row && gx >= 0 && gx < g.W) v = fa::stage_z(__ldg(row + gx), P.nodata);
      zw[WB::zidx(ly, lx)] = v;
    }
  }
}

// one in-block cell's D8 -> code + successor word
template <class S>
__device__ __forceinline__ void d8_put(S& s, int ly, int lx, int d, uint32_t forb) {
  using WB = typename S::WB;
  constexpr int R = S::RR;
  s.dirh[WB::hidx(ly, lx)] = (uint8_t)(d == kNoData ? kNoData : (d & 15));
  s.sb[ly * WB::BC + lx] = (uint8_t)succ_byte(d, forb);
}

// D8 down each column with a rolling 3x3 window (codes + successor words)
template <class S>
__device__ __forceinline__ void d8_block(S& s, int h, int w) {
  using WB = typename S::WB;
  const int lx = lane_id();
  if (lx >= w) return;
  const float* z = s.zwin();
  const uint32_t fc = forb_col(lx, w);
  int zi = WB::zidx(-1, lx);
  float u0 = z[zi - 1], u1 = z[zi], u2 = z[zi + 1];
  zi += WB::ZS;
  float c0 = z[zi - 1], c1 = z[zi], c2 = z[zi + 1];
  if (h == WB::BR) {
#pragma unroll 4
    for (int ly = 0; ly < WB::BR; ++ly) {
      zi += WB::ZS;
      const float e0 = z[zi - 1], e1 = z[zi], e2 = z[zi + 1];
      d8_put(s, ly, lx, d8_window(c1, u1, u2, c2, e2, e1, e0, c0, u0), fc | forb_row(ly, WB::BR));
      u0 = c0; u1 = c1; u2 = c2;
      c0 = e0; c1 = e1; c2 = e2;
    }
  } else {
    for (int ly = 0; ly < h; ++ly) {
      zi += WB::ZS;
      const float e0 = z[zi - 1], e1 = z[zi], e2 = z[zi + 1];
      d8_put(s, ly, lx, d8_window(c1, u1, u2, c2, e2, e1, e0, c0, u0), fc | forb_row(ly, h));
      u0 = c0; u1 = c1; u2 = c2;
      c0 = e0; c1 = e1; c2 = e2;
    }
  }
}

// ring cells around the block: NoData-ness into dirh (255 NoData / off-grid,
// 254 data) and, from their D8, which perimeter cells are entries.  A ring
// cell whose 3x3 window reaches a row this rank does not hold (beyond a strip
// halo row) has an unknown code: all its in-block neighbours count as entries.
template <class T, int WK, class S>
__device__ __forceinline__ void ring_entries(S& s, const PassArgs<T, WK>& P, int64_t y0, int h, int w) {
  using WB = typename S::WB;
  const float* z = s.zwin();
  const int rn = 2 * (w + 2) + 2 * h;
  for (int i = lane_id(); i < rn; i += 32) {
    int ly, lx;
    if (i < w + 2) { ly = -1; lx = i - 1; }
    else if (i < 2 * (w + 2)) { ly = h; lx = i - (w + 2) - 1; }
    else { const int j = i - 2 * (w + 2); ly = j >> 1; lx = (j & 1) ? w : -1; }
    const int zi = WB::zidx(ly, lx);
    const bool nd = isnan(z[zi]);
    s.dirh[WB::hidx(ly, lx)] = nd ? kNoData : kOut;
    if (nd) continue;
    const int64_t gy = y0 + ly;
    const bool unknown = (gy == -1 && P.dem_up) || (gy == P.g.H && P.dem_dn);
    uint32_t ks;  // codes whose target is marked
    if (unknown) {
      ks = 0x1FEu;
    } else {
      const int d = d8_window(z[zi], z[zi - WB::ZS], z[zi - WB::ZS + 1], z[zi + 1], z[zi + WB::ZS + 1],
                              z[zi + WB::ZS], z[zi + WB::ZS - 1], z[zi - 1], z[zi - WB::ZS - 1]);
      ks = (d >= 1 && d <= 8) ? (1u << d) : 0u;  // an outlet fallback (| 16) drains into NoData
    }
    while (ks) {
      const int k = __ffs(ks) - 1;
      ks &= ks - 1;
      const int ty = ly + dir_dy(k), tx = lx + dir_dx(k);
      if ((unsigned)ty < (unsigned)h && (unsigned)tx < (unsigned)w) need_inc(s.need, bperim_index(tx, ty, h, w));
    }
  }
}

// directions from global (pass 2 and pass 1 from dirs) + halo ring; bad
// codes -> NoData, flagged when `check`; with `entries`, ring codes that
// point into the block mark entry slots
template <class S>
__device__ __forceinline__ void load_dirs(S& s, const uint8_t* dirs, const uint8_t* dirs_up,
                                          const uint8_t* dirs_dn, const Geom& g, int64_t y0, int64_t x0, int h,
                                          int w, bool check, bool entries, uint32_t* status) {
  using WB = typename S::WB;
  const int lane = lane_id();
  const bool vec = w == WB::BC && ((x0 & 15) == 0) && ((g.W & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(dirs) & 15) == 0);
  bool bad = false;
  if (vec) {
    for (int q = lane; q < h * 2; q += 32) {
      const int ly = q >> 1, lx = (q & 1) * 16;
      uint4 v = __ldg(reinterpret_cast<const uint4*>(dirs + (y0 + ly) * g.W + x0 + lx));
      uint32_t* vv = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        // bytes > 8 and != 255 are illegal (D1)
        const uint32_t hi = __vcmpgtu4(vv[j], 0x08080808u) & ~__vcmpeq4(vv[j], 0xFFFFFFFFu);
        if (hi) { bad = true; vv[j] |= hi; }
      }
      uint32_t* dst = reinterpret_cast<uint32_t*>(&s.dirh[WB::hidx(ly, lx)]);
      dst[0] = vv[0];
      dst[1] = vv[1];
      dst[2] = vv[2];
      dst[3] = vv[3];
    }
  } else {
    for (int i = lane; i < h * WB::BC; i += 32) {
      const int ly = i >> 5, lx = i & 31;
      if (lx >= w) continue;
      uint8_t d = dirs[(y0 + ly) * g.W + x0 + lx];
      if (d > 8 && d != kNoData) { bad = true; d = kNoData; }
      s.dirh[WB::hidx(ly, lx)] = d;
    }
  }
  if (check && bad) atomicOr(status, ST_BADCODE);
  // ring codes -> dirh (data ring cells 254, NoData / off-grid 255); entries
  // count their outside donors
  auto ring_cell = [&](int ly, int lx, int code) {
    s.dirh[WB::hidx(ly, lx)] = code == kNoData ? kNoData : kOut;
    if (entries && code >= 1 && code <= 8) {
      const int ty = ly + dir_dy(code), tx = lx + dir_dx(code);
      if ((unsigned)ty < (unsigned)h && (unsigned)tx < (unsigned)w) need_inc(s.need, bperim_index(tx, ty, h, w));
    }
  };
  if (WB::BR == 32 && w == WB::BC && h == WB::BR) {
    // full block: the top and bottom ring rows are one coalesced byte per
    // lane, the side columns one byte per lane and row, corners on lanes 0-3
    const int64_t gu = y0 - 1, gd = y0 + h;
    const uint8_t* ru = gu < 0 ? dirs_up : gu >= g.H ? dirs_dn : dirs + gu * g.W;
    const uint8_t* rd = gd < 0 ? dirs_up : gd >= g.H ? dirs_dn : dirs + gd * g.W;
    const bool lok = x0 > 0, rok = x0 + WB::BC < g.W;
    const int cu = ru ? ru[x0 + lane] : kNoData, cd = rd ? rd[x0 + lane] : kNoData;
    const uint8_t* rl = dirs + (y0 + lane) * g.W;
    const int cl = lok ? rl[x0 - 1] : kNoData, cr = rok ? rl[x0 + WB::BC] : kNoData;
    int cc = kNoData, cy = -1, cx = -1;  // corners
    if (lane < 4) {
      cy = (lane & 1) ? h : -1;
      cx = (lane & 2) ? WB::BC : -1;
      const uint8_t* rc = (lane & 1) ? rd : ru;
      const bool ok = (lane & 2) ? rok : lok;
      if (rc && ok) cc = rc[x0 + cx];
    }
    ring_cell(-1, lane, cu);
    ring_cell(h, lane, cd);
    ring_cell(lane, -1, cl);
    ring_cell(lane, WB::BC, cr);
    if (lane < 4) ring_cell(cy, cx, cc);
    return;
  }
  const int rn = 2 * (w + 2) + 2 * h;
  for (int i = lane; i < rn; i += 32) {
    int ly, lx;
    if (i < w + 2) { ly = -1; lx = i - 1; }
    else if (i < 2 * (w + 2)) { ly = h; lx = i - (w + 2) - 1; }
    else { const int j = i - 2 * (w + 2); ly = j >> 1; lx = (j & 1) ? w : -1; }
    const int64_t gy = y0 + ly, gx = x0 + lx;
    int code = kNoData;
    if (gx >= 0 && gx < g.W && gy >= -1 && gy <= g.H) {
      const uint8_t* row = gy < 0 ? dirs_up : gy >= g.H ? dirs_dn : dirs + gy * g.W;
      if (row) code = row[gx];
    }
    s.dirh[WB::hidx(ly, lx)] = code == kNoData ? kNoData : kOut;
    if (entries && code >= 1 && code <= 8) {
      const int ty = ly + dir_dy(code), tx = lx + dir_dx(code);
      if ((unsigned)ty < (unsigned)h && (unsigned)tx < (unsigned)w) need_inc(s.need, bperim_index(tx, ty, h, w));
    }
  }
}


// ---------------------------------------------------------------- H2
// Donor masks of the 4 cells of dirh word hw: bit k-1 of byte j set iff the
// neighbour of cell j in direction k drains into it (its code is opp(k)).
template <int R>
__device__ __forceinline__ uint32_t donor_masks(const uint32_t* D, int hw) {
  constexpr int RW = WBT<R>::HS / 4;
  const uint32_t u0 = D[hw - RW - 1], u1 = D[hw - RW], u2 = D[hw - RW + 1];
  const uint32_t c0 = D[hw - 1], c1 = D[hw], c2 = D[hw + 1];
  const uint32_t d0 = D[hw + RW - 1], d1 = D[hw + RW], d2 = D[hw + RW + 1];
  const uint32_t nN = u1, nS = d1;
  const uint32_t nE = __funnelshift_r(c1, c2, 8), nW = __funnelshift_r(c0, c1, 24);
  const uint32_t nNE = __funnelshift_r(u1, u2, 8), nNW = __funnelshift_r(u0, u1, 24);
  const uint32_t nSE = __funnelshift_r(d1, d2, 8), nSW = __funnelshift_r(d0, d1, 24);
  // byte j of eq(n, c): bit 7 set iff byte j of n equals c (c < 0x80).  Exact
  // zero-byte test of n ^ c: the low 7 bits of a byte are non-zero iff adding
  // 0x7F sets its bit 7 (no carry between bytes), and bit 7 of n ^ c is bit 7
  // of n (codes 0..8, ring 254 / 255).  4 ops instead of __vcmpeq4's 7.
  auto eq7 = [](uint32_t n, uint32_t c) {
    const uint32_t y = ((n ^ c) & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;
    return ~(y | n) & 0x80808080u;
  };
  uint32_t m = eq7(nN, 0x05050505u) >> 7;
  m |= eq7(nNE, 0x06060606u) >> 6;
  m |= eq7(nE, 0x07070707u) >> 5;
  m |= eq7(nSE, 0x08080808u) >> 4;
  m |= eq7(nS, 0x01010101u) >> 3;
  m |= eq7(nSW, 0x02020202u) >> 2;
  m |= eq7(nW, 0x03030303u) >> 1;
  m |= eq7(nNW, 0x04040404u);
  return m;
}

// Donor masks by an 8-neighbour gather, 4 cells per 32-bit SWAR word (no
// atomics; Alg. 1 first loop P:L131-148) and the ready queue seeded with the
// sources (data cells without in-block donors).  The pending counts D(p)
// (Alg. 1 "dependencies") are the per-byte popcounts of the masks.  Returns
// this lane's data-cell count; by reference, the number of sources (warp
// total).  Ring codes (254/255) never equal a direction, so no bounds tests.
// With SUCC the successor words are computed here too, 4 cells at a time:
// the offsets of the codes come from a byte-permute table lookup (biased to
// bytes, zero-extended into 16-bit lanes) added with 16-bit SIMD adds; words
// on the block border take the scalar path (a code may leave the block
// there).  A cell draining into in-block NoData gets STOP afterwards, from
// the NoData cell's own donor mask (D8: that flow is dropped).
template <bool SUCC, class S>
__device__ __forceinline__ int build_masks(S& s, uint32_t& nsrc, int h, int w) {
  using WB = typename S::WB;
  constexpr int R = S::RR;
  constexpr int NQ = WB::BN / 128;  // words per lane
  static_assert(NQ <= 16, "source bits: 4 per word, 64 per lane");
  using SrcBits = typename std::conditional<(NQ > 8), unsigned long long, uint32_t>::type;
  const int lane = lane_id();
  const uint32_t* D = reinterpret_cast<const uint32_t*>(s.dirh);
  int ndata = 0;
  SrcBits srcbits = 0;
  uint32_t ndbits = 0;
#pragma unroll 1
  for (int k = 0; k < NQ; ++k) {
    const int q = k * 32 + lane;  // word: row q/8, cells 4(q%8)..+3
    const int ly = q >> 3, lx0 = (q & 7) * 4;
    const int hw = WB::hidx(ly, lx0) >> 2;
    const uint32_t c1 = D[hw];
    uint32_t m = donor_masks<R>(D, hw);
    // NoData (255) and cells outside a ragged block (254/255) are not cells
    const uint32_t nd = __vcmpgeu4(c1, 0xFEFEFEFEu);
    // in-block NoData cells with in-block donors: their donors are stopped below
    const uint32_t inb = ly >= h ? 0u : lx0 + 4 <= w ? 0xFFFFFFFFu : lx0 >= w ? 0u : (0xFFFFFFFFu >> (8 * (lx0 + 4 - w)));
    const uint32_t sink = SUCC ? (nd & inb & ~__vcmpeq4(m, 0u)) : 0u;
    m &= ~nd;
    // per-byte popcount of the masks, packed to 4 bits per cell
    uint32_t cnt = m - ((m >> 1) & 0x55555555u);
    cnt = (cnt & 0x33333333u) + ((cnt >> 2) & 0x33333333u);
    cnt = (cnt + (cnt >> 4)) & 0x0F0F0F0Fu;
#if FA_PEND_BYTES
    s.pend[q] = cnt;
#else
    reinterpret_cast<uint16_t*>(s.pend)[q] =
        (uint16_t)((cnt & 0xFu) | ((cnt >> 4) & 0xF0u) | ((cnt >> 8) & 0xF00u) | ((cnt >> 12) & 0xF000u));
#endif
    ndbits |= (sink ? 1u : 0u) << k;
    ndata += 4 - (__popc(nd) >> 3);
    if constexpr (SUCC) {
      uint32_t sbw;
      if (h == WB::BR && w == WB::BC) {
        // full block: the successor bytes are the codes themselves, plus
        // SB_EXIT on the block border -- a per-byte lookup (selector = code
        // - 1) of the codes that leave the block through that side
        const uint32_t nib = code_nibbles(c1);
        sbw = sb_word(c1, nib, border_exits<WB::BR>(nib, ly, lx0));
      } else {
        sbw = 0u;
        const uint32_t fr = forb_row(ly, h);
#pragma unroll
        for (int j = 0; j < 4; ++j) sbw |= succ_byte((c1 >> (8 * j)) & 0xFF, fr | forb_col(lx0 + j, w)) << (8 * j);
      }
      reinterpret_cast<uint32_t*>(s.sb)[q] = sbw;
    }
    const uint32_t src4 = __vcmpeq4(m, 0u) & ~nd & 0x80808080u;  // sources: bit 7 of each byte
    srcbits |= (SrcBits)(((src4 >> 7) & 1u) | ((src4 >> 14) & 2u) | ((src4 >> 21) & 4u) | ((src4 >> 28) & 8u))
               << (4 * k);
  }
  if constexpr (SUCC) {
    // donors of in-block NoData cells: their flow is dropped (STOP)
    __syncwarp();
#pragma unroll 1
    for (int k = 0; k < NQ; ++k) {
      if (!((ndbits >> k) & 1u)) continue;
      const int q = k * 32 + lane;
      const int hw = WB::hidx(q >> 3, (q & 7) * 4) >> 2;
      const uint32_t pw = donor_masks<R>(D, hw);  // raw masks (the NoData cells' too)
      const int ly = q >> 3, lx0 = (q & 7) * 4;
      const uint32_t inb = ly >= h ? 0u : lx0 + 4 <= w ? 0xFFFFFFFFu : lx0 >= w ? 0u : (0xFFFFFFFFu >> (8 * (lx0 + 4 - w)));
      const uint32_t nd = __vcmpgeu4(D[hw], 0xFEFEFEFEu) & inb;  // in-block NoData only (not the ring)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (!((nd >> (8 * j)) & 1u)) continue;
        uint32_t mm = (pw >> (8 * j)) & 0xFFu;
        while (mm) {
          const int kk = __ffs(mm);
          mm &= mm - 1;
          s.sb[4 * q + j + WB::offA(kk)] = (uint8_t)(SB_STOP | SB_DROP);
        }
      }
    }
  }
  // compact: exclusive scan of the per-lane counts, then each lane writes its cells
  const int cnt = sizeof(SrcBits) == 8 ? __popcll((unsigned long long)srcbits) : __popc((uint32_t)srcbits);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += v;
  }
  nsrc = (uint32_t)__shfl_sync(kFull, incl, 31);
  int pos = incl - cnt;
  while (srcbits) {
    const int bpos = sizeof(SrcBits) == 8 ? __ffsll((long long)srcbits) - 1 : __ffs((int)srcbits) - 1;
    srcbits &= srcbits - 1;
    const int k = bpos >> 2, j = bpos & 3;
    FA_CHECK(pos < WB::BN);
    s.src[pos++] = (uint16_t)(4 * (k * 32 + lane) + j);
  }
  return ndata;
}

// ---------------------------------------------------------------- H3
// Alg. 1 queue loop (see the file comment).  On entry succ, pend and the
// queue (sources) are set and A (= w [+ x]) is in the block's rows of acc,
// all visible to the warp.  Returns the number of cells popped (retired;
// warp-uniform).
// fire-and-forget reduction into global memory (explicit .global: the
// addresses come from elt(), whose state space the compiler cannot see)
template <class T>
__device__ __forceinline__ void g_add(T* p, T v);
template <>
__device__ __forceinline__ void g_add<double>(double* p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v));
}
template <>
__device__ __forceinline__ void g_add<uint32_t>(uint32_t* p, uint32_t v) {
  asm volatile("red.global.add.u32 [%0], %1;" ::"l"(p), "r"(v));
}
template <>
__device__ __forceinline__ void g_add<unsigned long long>(unsigned long long* p, unsigned long long v) {
  asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(v));
}
// &base[i] for a 32-bit element offset as ONE wide multiply-add (the
// compiler otherwise splits the block's base into a uniform pointer and a
// 64-bit offset and rebuilds the sum with 4 instructions per access)
template <class T>
__device__ __forceinline__ T* elt(T* base, uint32_t i) {
  T* r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(i), "n"((int)sizeof(T)), "l"(base));
  return r;
}
// element offset of block cell c = 32*ly + lx in rows of stride 32 + wm
__device__ __forceinline__ uint32_t cell_off(uint32_t c, uint32_t wm) { return c + (c >> 5) * wm; }

// Tail of Alg. 1's queue loop with chain bursts.  When few cells are ready
// the block is working through its long in-block chains, one L2 round trip
// per cell.  A successor whose only pending donor is the lane's own cell
// (count 1 at the start of the iteration) is final as soon as that cell is:
// A(succ) already holds w plus every earlier donor, so the lane follows the
// chain up to K cells per iteration with all K loads in flight at once and
// writes the values with plain stores.  Junction successors (count > 1) take
// the RED + shared-count path and are queued by the lane that takes the
// count to zero.  Counts are read in phase 1 and decremented in phase 2,
// separated by __syncwarp, so every chain decision sees the counts of the
// iteration start (no other lane can push into a chain cell: its one pending
// donor is the lane's own cell).  Returns the number of cells processed.
template <int K, class T, int R, bool Z>
__device__ __forceinline__ uint32_t kahn_chain_tail(WSmem<T, R, Z>& s, uint32_t head, uint32_t tail, T* Ab,
                                                    int64_t W) {
  const int lane = lane_id();
  const unsigned lt = (1u << lane) - 1u;
  uint16_t* Q = s.src;
  const uint32_t wm = (uint32_t)W - 32u;
  uint32_t done = 0;
  int c = -1;          // the lane's cell (its value a is final once loaded)
  bool fresh = false;  // c was just taken from the queue: a must be loaded
  T a = (T)0;
  for (;;) {
    __syncwarp();
    const unsigned idle = __ballot_sync(kFull, c < 0);
    const uint32_t avail = tail - head;
    if (idle == kFull && avail == 0u) break;
    if (c < 0) {
      const uint32_t r = (uint32_t)__popc(idle & lt);
      if (r < avail) {
        FA_CHECK(head + r < (uint32_t)WSmem<T, R, Z>::WB::BN);
        c = Q[head + r];
        fresh = true;
      }
    }
    head += min((uint32_t)__popc(idle), avail);
    // phase 1: the chain ahead of c
    uint32_t cc[K];
    uint32_t cur = (uint32_t)c, end_t = 0u;
    bool end_ok = false;  // the chain ends at a junction target end_t (else at a stop)
    int n = 0;
    bool go = c >= 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      cc[k] = 0u;
      if (go) {
        const uint32_t sbv = s.sb[cur];
        const bool ok = sb_go(sbv);
        const uint32_t t = ok ? WBT<R>::target(cur, sbv) : 0u;
        FA_CHECK(t < (uint32_t)WBT<R>::BN);
        go = ok && pend_get(s.pend, t) == 1u;
        if (go) {
          cc[k] = t;
          cur = t;
          n = k + 1;
        } else {
          end_ok = ok;
          end_t = t;
        }
      }
    }
    __syncwarp();
    // phase 2: one round of loads, the chain's prefix sums, then the junction push
    uint32_t ready = 0u, t = 0u;
    if (c >= 0) {
      T x[K];
      T* pk[K];
      if (fresh) a = __ldcg(elt(Ab, cell_off((uint32_t)c, wm)));
#pragma unroll
      for (int k = 0; k < K; ++k) {
        pk[k] = elt(Ab, cell_off(cc[k], wm));
        if (k < n) x[k] = __ldcg(pk[k]);
      }
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (k < n) {
          a += x[k];
          *pk[k] = a;
        }
      done += (fresh ? 1u : 0u) + (uint32_t)n;
      fresh = false;
      if (go) {
        c = (int)cur;  // the chain goes on: continue from its last cell next iteration
      } else {
        c = -1;
        if (end_ok) {
          // "A(n) <- A(n) + A(c)", "decrement D(n)" (Alg. 1)
          t = end_t;
          g_add(elt(Ab, cell_off(t, wm)), a);
          ready = pend_dec(s.pend, t);
        }
      }
    }
    const unsigned bm = __ballot_sync(kFull, ready != 0u);
    FA_CHECK(!ready || (t < (uint32_t)WBT<R>::BN && tail + (uint32_t)__popc(bm & lt) < (uint32_t)WBT<R>::BN));
    if (ready) Q[tail + (uint32_t)__popc(bm & lt)] = (uint16_t)t;
    tail += (uint32_t)__popc(bm);
  }
  __syncwarp();
  return __reduce_add_sync(kFull, done);
}

template <class T, int R, bool Z, bool ABS = false>
__device__ __forceinline__ uint32_t kahn_block(WSmem<T, R, Z>& s, uint32_t nsrc, T* Ab, int64_t W,
                                               const float* Alb = nullptr) {
  const int lane = lane_id();
  const unsigned lt = (1u << lane) - 1u;
  uint16_t* Q = s.src;
  // element offset of block cell c = 32*ly + lx in the raster rows: c + ly*(W-32)
  const uint32_t wm = (uint32_t)W - 32u;
  uint32_t head = 0, tail = nsrc;
  while (head < tail) {
#if FA_CHAIN_TAIL
    // the queue has narrowed to the block's long in-block chains: finish
    // with chain bursts (kahn_chain_tail), which carry values along chains
    // instead of one L2 round trip per cell
    if constexpr (!ABS) {
      if (tail - head < FA_CHAIN_TAIL) {
        __syncwarp();
        return head + kahn_chain_tail<FA_CHAIN_K>(s, head, tail, Ab, W);
      }
    }
#endif
    __syncwarp();
    const uint32_t q = head + (uint32_t)lane;
    const bool valid = q < tail;
    head = tail - head < 32u ? tail : head + 32u;
    uint32_t ready = 0, t = 0;
    if (valid) {
      const uint32_t c = Q[q];
      const uint32_t sbv = s.sb[c];
      if (sb_go(sbv)) {
        // "A(n) <- A(n) + A(c)" and "decrement D(n)" (Alg. 1);
        // A(c) is final: every donor of c was popped in an earlier iteration
        t = WBT<R>::target(c, sbv);
        FA_CHECK(c < (uint32_t)WBT<R>::BN && t < (uint32_t)WBT<R>::BN);
        T a = __ldcg(elt(Ab, cell_off(c, wm)));
        if constexpr (ABS) a *= (T)__ldg(Alb + (c + (c >> 5) * wm));  // "alpha(n) A(n)"
        g_add(elt(Ab, cell_off(t, wm)), a);
        ready = pend_dec(s.pend, t);  // the last pending donor: n joins the queue
      }
    }
    const unsigned bm = __ballot_sync(kFull, ready != 0u);
    FA_CHECK(!ready || (t < (uint32_t)WBT<R>::BN && tail + (uint32_t)__popc(bm & lt) < (uint32_t)WBT<R>::BN));
    if (ready) Q[tail + (uint32_t)__popc(bm & lt)] = (uint16_t)t;
    tail += (uint32_t)__popc(bm);
  }
  __syncwarp();
  return tail;
}

// ---------------------------------------------------------------- values
// A = w (Eq. 1; Alg. 1 "A(c) <- A(c) + 1") in the block's rows of
// acc, NoData cells get the marker (D9); returns Σw over data cells (integer
// weights; the u32 overflow check, D10)
template <class T, int R, bool Z, int WK>
__device__ __forceinline__ unsigned long long init_values(WSmem<T, R, Z>& s, const void* wp, const Geom& g,
                                                          int64_t y0, int64_t x0, int h, int w, T* out,
                                                          uint32_t* status) {
  using WB = WBT<R>;
  const int lane = lane_id();
  unsigned long long wsum = 0;
  bool bad = false;
  const bool vec = w == WB::BC && ((x0 & 3) == 0) && ((g.W & 3) == 0) &&
                   (WK == 0 || (reinterpret_cast<uintptr_t>(wp) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  // the block's first cell in w and out; cell offsets ly * W + lx in 32 bits
  // (as in the queue loop), one wide multiply-add per access
  const uint32_t* Wb = static_cast<const uint32_t*>(wp) + (WK != 0 ? y0 * g.W + x0 : 0);
  T* ob = out + y0 * g.W + x0;
  const uint32_t WW = (uint32_t)g.W;
  for (int q = lane; q < h * (WB::BC / 4); q += 32) {
    const int ly = q >> 3, lx = (q & 7) * 4;
    const uint32_t dw = *reinterpret_cast<const uint32_t*>(&s.dirh[WB::hidx(ly, lx)]);
    const uint32_t off = (uint32_t)ly * WW + (uint32_t)lx;
    // NoData (255) or cells right of a ragged block (255): the rare path
    const bool anynd = (dw & 0x80808080u) != 0u;
    uint32_t u[4] = {1u, 1u, 1u, 1u};
    if (WK != 0) {
      if (vec) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(elt(Wb, off)));
        u[0] = v.x; u[1] = v.y; u[2] = v.z; u[3] = v.w;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (lx + j < w) u[j] = __ldg(elt(Wb, off + j));
      }
    }
    alignas(16) T v[4];
    uint32_t badw = 0;  // f32 weights failing weight_ok, data or not (checked below)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if constexpr (WK == 0) {
        v[j] = (T)1;
      } else if constexpr (WK == 1) {
        v[j] = (T)u[j];
        if (((dw >> (8 * j)) & 0xFF) < kOut) wsum += u[j];
      } else {
        // weight_ok on the bits (D21): finite and >= 0 is u <= 0x7F7FFFFF or -0
        badw |= (uint32_t)((u[j] > 0x7F7FFFFFu) & (u[j] != 0x80000000u)) << j;
        v[j] = (T)__uint_as_float(u[j]);
      }
    }
    if (anynd) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (((dw >> (8 * j)) & 0xFF) == kNoData) {
          v[j] = AccT<T>::marker();
          badw &= ~(1u << j);  // NoData weights are ignored
        }
    }
    if (badw) bad = true;
    if (vec) {
      if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<uint4*>(elt(ob, off)) = *reinterpret_cast<const uint4*>(v);
      } else {
        uint4* o = reinterpret_cast<uint4*>(elt(ob, off));
        o[0] = *reinterpret_cast<const uint4*>(&v[0]);
        o[1] = *reinterpret_cast<const uint4*>(&v[2]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (lx + j < w) *elt(ob, off + j) = v[j];
    }
  }
  if (bad) atomicOr(status, ST_BADWEIGHT);
  return wsum;
}

// the block's D8 codes to global (16-byte rows when aligned)
template <class S>
__device__ __forceinline__ void write_dirs(const S& s, uint8_t* dirs, const Geom& g, int64_t y0, int64_t x0, int h,
                                           int w) {
  using WB = typename S::WB;
  const int lane = lane_id();
  const bool vec = w == WB::BC && ((x0 & 15) == 0) && ((g.W & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(dirs) & 15) == 0);
  if (vec) {
    for (int q = lane; q < h * 2; q += 32) {
      const int ly = q >> 1, lx = (q & 1) * 16;
      const uint32_t* src = reinterpret_cast<const uint32_t*>(&s.dirh[WB::hidx(ly, lx)]);
      *reinterpret_cast<uint4*>(dirs + (y0 + ly) * g.W + x0 + lx) = make_uint4(src[0], src[1], src[2], src[3]);
    }
  } else {
    for (int i = lane; i < h * WB::BC; i += 32) {
      const int ly = i >> 5, lx = i & 31;
      if (lx < w) dirs[(y0 + ly) * g.W + x0 + lx] = s.dirh[WB::hidx(ly, lx)];
    }
  }
}

// ---------------------------------------------------------------- H4
// Alg. 2 FollowPath from the perimeter cells that need their
// exit (entries -- cells a ring cell drains into -- and, in tile-records mode,
// every slot on a tile edge), then the block exits.  An exit's child count in
// the block-exit graph is the number of outside donors over the entries whose
// path reaches it; an exit with none (a leaf: ~75 % of exits on cfg3) has its
// final value already, so outside tile-records mode it is not a graph node:
// its value goes straight into the offset of its target slot (x_slot, the
// entry's external inbound flow, D11).  Other exits become nodes (compacted,
// one global atomic per warp).  slot_root[entry] = node of its exit.  Lane l
// handles slots l, l+32, l+64, l+96.
template <class T, int R, class S, int WK, bool ABS = false>
__device__ __forceinline__ void block_records(S& s, const PassArgs<T, WK>& P, int64_t b, int64_t y0,
                                              int64_t x0, int h, int w) {
  using WB = WBT<R>;
  constexpr int NJ = WB::NJ;
  constexpr uint32_t kNoP = 0xFFu;
  const Geom& g = P.g;
  const int lane = lane_id();
  const unsigned lt = (1u << lane) - 1u;
  // absorption: alpha of block cell c (same row-major layout as acc)
  const float* Alb = ABS ? P.alpha + y0 * g.W + x0 : nullptr;
  const uint32_t wmA = (uint32_t)g.W - 32u;
  auto alpha_of = [&](int c) -> T { return (T)__ldg(Alb + ((uint32_t)c + ((uint32_t)c >> 5) * wmA)); };
  const int np = bperim_count(h, w);
  uint32_t* slot_nid = s.slot_nid();  // the queue is dead after the queue loop
  uint32_t* nchild = slot_nid + WB::NP;  // per exit slot: outside donors of the entries draining to it
  for (int i = lane; i < WB::NP; i += 32) nchild[i] = 0u;
  // the block's tile: only tile-records mode (cut) uses tile edges and the
  // out-of-tile flag (two integer divisions saved per block otherwise)
  int64_t t0y = 0, t0x = 0, th = 0, tw = 0;
  if (P.cut) g.tile_box(g.tile_of_block(b), t0y, t0x, th, tw);
  int cell[NJ];
  bool ex[NJ], want[NJ], tedge[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int p = lane + 32 * j;
    cell[j] = -1;
    ex[j] = want[j] = tedge[j] = false;
    if (p < np) {
      int px, py;
      bperim_xy(p, h, w, px, py);
      cell[j] = py * WB::BC + px;
      const bool data = s.dirh[WB::hidx(py, px)] != kNoData;
      ex[j] = data && sb_exit(s.sb[cell[j]]);
      if (P.cut) {  // tile records: every slot on a tile edge needs its link
        const int64_t gy = y0 + py, gx = x0 + px;
        tedge[j] = gy == t0y || gx == t0x || gy == t0y + th - 1 || gx == t0x + tw - 1;
      }
      want[j] = data && !ex[j] && (s.need[p] != 0u || tedge[j]);
    }
    // path products start at 1 (exits that are entries keep it: no cell before the exit)
    if (ABS && p < WB::PB) P.slot_f[b * WB::PB + p] = (T)1;
  }
  __syncwarp();
  // exits that are entries themselves count their own outside donors
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int p = lane + 32 * j;
    if (ex[j] && s.need[p]) atomicAdd(&nchild[p], (uint32_t)s.need[p]);
  }
  // walks (lanes refill from a warp-uniform work list as they finish); the
  // root (exit slot or kNoP) of a walked slot p is kept in need[p] afterwards
  uint32_t wl[NJ];
  int nwalk = 0;
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    wl[j] = __ballot_sync(kFull, want[j]);
    nwalk += __popc(wl[j]);
  }
  int head = 0;
  int p = -1, c = 0;
  uint32_t sbv = SB_STOP;  // successor byte of the walk's cell
  T f = (T)1;  // absorption: product of alpha along the walked path so far
  for (;;) {
    const unsigned idle = __ballot_sync(kFull, p < 0);
    if (idle == kFull && head >= nwalk) break;
    if (p < 0) {
      const int r = head + __popc(idle & lt);
      if (r < nwalk) {
        // r-th wanted slot: the rr-th set bit of wl[j]
        int j = 0, rr = r;
        uint32_t m = wl[0];
#pragma unroll
        for (int jj = 1; jj < NJ; ++jj) {
          const int c0 = __popc(m);
          if (j == jj - 1 && rr >= c0) {
            j = jj;
            rr -= c0;
            m = wl[jj];
          }
        }
        const int l = __fns(m, 0, rr + 1);
        p = l + 32 * j;
        int px, py;
        bperim_xy(p, h, w, px, py);
        c = py * WB::BC + px;
        sbv = s.sb[c];
        f = (T)1;
      }
    }
    head += __popc(idle);
    if (p < 0) continue;
    if (!sb_go(sbv)) {
      if (ABS) P.slot_f[b * WB::PB + p] = f;  // the entry's offset reaches its exit scaled by f
      uint32_t rp = kNoP;
      if (sb_exit(sbv)) {
        rp = (uint32_t)bperim_index(c & 31, c >> 5, h, w);
        // tile-records mode: an exit reached from a tile-edge slot is a node too
        const uint32_t k = s.need[p] ? s.need[p] : (P.cut ? 1u : 0u);
        FA_CHECK(rp < 128u);
        if (k) atomicAdd(&nchild[rp], k);
      }
      s.need[p] = (uint8_t)rp;  // only this lane touches need[p] from here on
      p = -1;
      continue;
    }
    if (ABS) f *= alpha_of(c);
    c = (int)WB::target((uint32_t)c, sbv);
    FA_CHECK((unsigned)c < (unsigned)WB::BN);
    sbv = s.sb[c];
#pragma unroll
    for (int u = 1; u < FA_REC_STEPS; ++u) {  // more steps per refill round
      if (!sb_go(sbv)) break;
      if (ABS) f *= alpha_of(c);
      c = (int)WB::target((uint32_t)c, sbv);
      sbv = s.sb[c];
    }
  }
  __syncwarp();
  // exits: leaves push their value to the target slot, the rest become nodes
  // (in tile-records mode also every exit leaving its tile: FlowExternal)
  bool node[NJ];
  uint8_t flg[NJ];
  int tyv[NJ], txv[NJ];
  int nex = 0;
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int p2 = lane + 32 * j;
    flg[j] = 0;
    tyv[j] = txv[j] = 0;
    if (ex[j]) {
      const int px = cell[j] & 31, py = cell[j] >> 5;
      const int d = s.dirh[WB::hidx(py, px)];
      tyv[j] = py + dir_dy(d);
      txv[j] = px + dir_dx(d);
      const bool dead = s.dirh[WB::hidx(tyv[j], txv[j])] == kNoData;
      const int64_t gy = y0 + tyv[j], gx = x0 + txv[j];
      flg[j] = dead ? NF_DEAD : 0;
      if (P.cut && (gy < t0y || gx < t0x || gy >= t0y + th || gx >= t0x + tw)) flg[j] |= NF_OUT_TILE;
    }
    node[j] = ex[j] && (nchild[p2] != 0u || (P.cut && ((flg[j] & NF_OUT_TILE) || tedge[j])));
    nex += __popc(__ballot_sync(kFull, node[j]));
  }
  uint32_t base = 0;
  if (lane == 0 && nex) base = atomicAdd(P.node_count, (uint32_t)nex);
  base = __shfl_sync(kFull, base, 0);
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int p2 = lane + 32 * j;
    const unsigned em = __ballot_sync(kFull, node[j]);
    uint32_t nid = kNone;
    if (ex[j]) {
      const int px = cell[j] & 31, py = cell[j] >> 5;
      const int ty = tyv[j], tx = txv[j];
      const uint8_t fl = flg[j];
      const bool dead = (fl & NF_DEAD) != 0;
      const int64_t gy = y0 + ty, gx = x0 + tx;
      uint32_t tgt = kNone;  // none: dropped, or in another strip (carried by the tile records)
      if (!dead && gy >= 0 && gy < g.H) {
        int64_t tb;
        int tly, tlx, bh, bw;
        if (g.regular) {
          // plain block grid: the target block is a neighbour of b
          const int dby = ty < 0 ? -1 : ty >= h ? 1 : 0, dbx = tx < 0 ? -1 : tx >= w ? 1 : 0;
          tb = b + (int64_t)dby * g.NBC + dbx;
          tly = ty - dby * WB::BR;
          tlx = tx - dbx * WB::BC;
          const int64_t ty0 = y0 + (int64_t)dby * WB::BR, tx0 = x0 + (int64_t)dbx * WB::BC;
          bh = (int)(g.H - ty0 < WB::BR ? g.H - ty0 : WB::BR);
          bw = (int)(g.W - tx0 < WB::BC ? g.W - tx0 : WB::BC);
        } else {
          tb = g.block_of(gy, gx, tly, tlx);
          int64_t by0, bx0;
          g.block_box(tb, by0, bx0, bh, bw);
        }
        tgt = (uint32_t)(tb * WB::PB + bperim_index(tlx, tly, bh, bw));
      }
      T a;
      if constexpr (S::kValues) a = s.a[cell[j]];  // the block's values are on chip
      else a = __ldcg(P.acc + (y0 + py) * g.W + x0 + px);
      if (node[j]) {
        nid = base + (uint32_t)__popc(em & lt);
        if (ABS) P.node_alpha[nid] = (float)alpha_of(cell[j]);
        FA_CHECK(nid < (uint32_t)(g.nblocks * WB::PB));
        P.node_val[nid] = a;
        P.node_slot[nid] = (uint32_t)(b * WB::PB + p2);
        P.node_tgt[nid] = tgt;
        P.node_flags[nid] = fl;
      } else if (tgt != kNone) {
        // a leaf: S(e) = A_B(e), nothing flows in from upstream blocks
        FA_CHECK(tgt < (uint32_t)(g.nblocks * WB::PB));
        atomic_add(&P.x_slot[tgt], ABS ? a * alpha_of(cell[j]) : a);
      }
    }
    if (p2 < WB::PB) slot_nid[p2] = nid;
    base += (uint32_t)__popc(em);
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int p2 = lane + 32 * j;
    if (p2 >= WB::PB) continue;
    uint32_t root = kNone;
    if (ex[j]) root = slot_nid[p2];
    else if (want[j] && s.need[p2] != kNoP) {
      FA_CHECK(s.need[p2] < WB::PB);
      root = slot_nid[s.need[p2]];
    }
    P.slot_root[b * WB::PB + p2] = root;
  }
}

// ---------------------------------------------------------------- pass 1
// FULL: every non-empty block of the launch is a whole R x 32 block (the
// raster, strip and tile sizes are multiples of the block shape): h and w
// are compile-time constants, the ragged-block paths compile out
template <class T, int R, int WK, bool FROM_DEM, bool ABS = false, bool FULL = false>
__global__ void __launch_bounds__(32 * kNW, FA_P1_MINB * 4 / kNW) k_pass1(PassArgs<T, WK> P) {
  using WB = WBT<R>;
  constexpr bool Z = FROM_DEM;
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  WSmem<T, R, Z>& s = reinterpret_cast<WSmem<T, R, Z>*>(smem)[warp];
  const Geom& g = P.g;
  const int lane = lane_id();
  // FA_P1_KPW blocks per warp, one after another (a CTA owns KPW * nw
  // consecutive blocks): a CTA slot is refilled KPW times less often
#if FA_P1_KPW > 1
#pragma unroll 1
  for (int it = 0; it < FA_P1_KPW; ++it) {
  if (it) __syncwarp();
  const int64_t b = P.b_begin + ((int64_t)blockIdx.x * FA_P1_KPW + it) * g.nw + warp;
  if (b >= P.b_end) return;
#else
  {
  const int64_t b = P.b_begin + (int64_t)blockIdx.x * g.nw + warp;
  if (b >= P.b_end) return;
#endif
  int64_t y0, x0;
  int h, w;
  g.block_box(b, y0, x0, h, w);
  if (h <= 0 || w <= 0) {
    for (int p = lane; p < WB::PB; p += 32) P.slot_root[b * WB::PB + p] = kNone;
#if FA_P1_KPW > 1
    continue;
#else
    return;
#endif
  }
  if constexpr (FULL) {
    h = WB::BR;
    w = WB::BC;
  }
#if FA_P1_PREFETCH & 1
  // the block's weight rows are read only after the codes are staged and the
  // donor masks built: start their DRAM reads now
  if (WK != 0 && lane < h) {
    const char* wrow = static_cast<const char*>(P.w) + ((y0 + lane) * g.W + x0) * 4;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(wrow));
  }
#endif
#if FA_P1_PREFETCH & 2
  // the entry offsets of the 4 neighbour blocks: the leaf exits' reductions
  // (block_records) land there
  {
    constexpr int LINES = (WB::PB * (int)sizeof(T) + 127) / 128;
    const int nb = lane / 8, ln = lane % 8;
    const int64_t tb = nb == 0 ? b - 1 : nb == 1 ? b + 1 : nb == 2 ? b - g.NBC : b + g.NBC;
    if (ln < LINES && tb >= 0 && tb < g.nblocks)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(P.x_slot + tb * WB::PB) + ln * 128));
  }
#endif
  init_smem(s);
  if (FROM_DEM) {
    stage_z(s, P, y0, x0, h, w);
    __syncwarp();
    d8_block(s, h, w);
    ring_entries(s, P, y0, h, w);
    __syncwarp();
    if (P.dirs_out) write_dirs(s, P.dirs_out, g, y0, x0, h, w);
  } else {
    __syncwarp();
    load_dirs(s, P.dirs_in, P.dirs_up, P.dirs_dn, g, y0, x0, h, w, true, true, P.status);
  }
  __syncwarp();
  uint32_t nsrc;
  const int ndata = build_masks<!FROM_DEM>(s, nsrc, h, w);
  // RETAIN: the block-local accumulation is computed in place in acc
  unsigned long long wsum = init_values<T, R, Z, WK>(s, P.w, g, y0, x0, h, w, P.acc, P.status);
  if constexpr (ABS) {
    // D21-like validation of alpha: data cells need a value in [0, 1]
    bool bad = false;
    for (int i = lane; i < h * WB::BC; i += 32) {
      const int ly = i >> 5, lx = i & 31;
      if (lx >= w || s.dirh[WB::hidx(ly, lx)] >= kOut) continue;
      const float al = __ldg(P.alpha + (y0 + ly) * g.W + x0 + lx);
      if (!(al >= 0.0f && al <= 1.0f)) bad = true;
    }
    if (__any_sync(kFull, bad) && lane == 0) atomicOr(P.status, ST_BADALPHA);
  }
  const uint32_t popped = kahn_block<T, R, Z, ABS>(s, nsrc, P.acc + y0 * g.W + x0, g.W,
                                                   ABS ? P.alpha + y0 * g.W + x0 : nullptr);
  const int tot_data = __reduce_add_sync(kFull, ndata);
  if (lane == 0 && (int)popped != tot_data) atomicOr(P.status, ST_CYCLE);  // a cell never became ready
  if (!std::is_same<T, double>::value && P.wsum) {
    if (WK == 0) wsum = lane == 0 ? (unsigned long long)tot_data : 0;
    for (int o = 16; o; o >>= 1) wsum += __shfl_xor_sync(kFull, wsum, o);
    if (lane == 0 && wsum) atomicAdd(P.wsum, wsum);
  }
  block_records<T, R, WSmem<T, R, Z>, WK, ABS>(s, P, b, y0, x0, h, w);
  }
}

// ---------------------------------------------------------------- pass 2
template <class T, int R, int WK>
__global__ void __launch_bounds__(32 * kNW) k_pass2(PassArgs<T, WK> P) {
  using WB = WBT<R>;
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  WSmem<T, R, false>& s = reinterpret_cast<WSmem<T, R, false>*>(smem)[warp];
  const Geom& g = P.g;
  const int64_t b = P.b_begin + (int64_t)blockIdx.x * g.nw + warp;
  if (b >= P.b_end) return;
  const int lane = lane_id();
  int64_t y0, x0;
  int h, w;
  g.block_box(b, y0, x0, h, w);
  if (h <= 0 || w <= 0) return;
  init_smem(s);
  __syncwarp();
  load_dirs(s, P.dirs_in, P.dirs_up, P.dirs_dn, g, y0, x0, h, w, false, false, P.status);
  __syncwarp();
  uint32_t nsrc;
  const int ndata = build_masks<true>(s, nsrc, h, w);
  init_values<T, R, false, WK>(s, P.w, g, y0, x0, h, w, P.acc, P.status);
  __syncwarp();
  // inject x at the block perimeter (offset propagation; D12)
  const int np = bperim_count(h, w);
  for (int p = lane; p < np; p += 32) {
    int px, py;
    bperim_xy(p, h, w, px, py);
    if (s.dirh[WB::hidx(py, px)] == kNoData) continue;
    T* a = P.acc + (y0 + py) * g.W + x0 + px;
    *a = *a + P.x_slot[b * WB::PB + p];
  }
  const uint32_t popped = kahn_block(s, nsrc, P.acc + y0 * g.W + x0, g.W);
  const int tot_data = __reduce_add_sync(kFull, ndata);
  if (lane == 0 && (int)popped != tot_data) atomicOr(P.status, ST_CYCLE);
}

// ---------------------------------------------------------------- pass 1 / pass 2, values on chip
// The block's values live in shared memory (VSmem, ~14 KB per warp for f64),
// so the whole of Alg. 1 runs without a global-memory round trip:
//   * in-block donor counts (one byte per cell) and successor words are
//     built by an 8-neighbour SWAR gather, 4 cells per 32-bit word (no
//     atomics; Alg. 1's first loop);
//   * A = w is staged once (coalesced), NoData cells get the marker;
//   * the queue of Alg. 1 becomes "the last donor continues": a
//     lane takes a source and pushes its value along its successors, adding
//     it into A(n) and decrementing n's count; when the count reaches zero
//     A(n) is final and the lane continues from n with the value in a
//     register; otherwise it takes the next source.  Two lanes pushing into
//     the same cell in one iteration are ordered through a claim byte (each
//     writes its lane, the one read back pushes, the others retry next
//     iteration) -- so every push is a plain read-modify-write of shared
//     memory (no atomics at all in the loop);
//   * visibility: every iteration starts with __syncwarp (memory ordering
//     among the warp's lanes), and within an iteration each cell's value and
//     count are touched by one lane only;
//   * the final values are written to the output once, coalesced (RETAIN);
//     with EVICT pass 1 writes nothing and pass 2 reruns the block with
//     w + x injected at its entries.
template <class T, int R>
struct __align__(16) VSmem {
  using WB = WBT<R>;
  using VT = T;
  static constexpr int RR = R;
  static constexpr bool kValues = true;
  // A(p): w(p) plus the pushes received so far.  With D8 fused the 2-cell
  // halo z window of the block lives here first (dead once the codes are made)
  static constexpr int NA = (int)((WB::BN * sizeof(T) > WB::ZN * sizeof(float) ? WB::BN * sizeof(T)
                                                                              : WB::ZN * sizeof(float)) / sizeof(T));
  T a[NA];
  __device__ __forceinline__ float* zwin() { return reinterpret_cast<float*>(a); }
  uint8_t dirh[WB::HN];            // codes + ring (as WSmem)
  alignas(16) uint8_t cnt[WB::BN];  // pending in-block donors, one byte per cell
  uint8_t claim[WB::BN];            // per iteration: the lane pushing into the cell
  alignas(8) uint8_t sb[WB::BN];   // successor bytes
  alignas(16) uint16_t src[WB::BN];  // sources (Alg. 1's initial queue); records scratch afterwards
  alignas(4) uint8_t need[WB::NP];
  __device__ __forceinline__ uint32_t* slot_nid() { return reinterpret_cast<uint32_t*>(src); }
  static_assert(WB::BN * 2 >= 2 * WB::NP * 4, "records scratch lives in the queue");
};

constexpr int kNWV = 2;  // warps (blocks) per CTA of the on-chip-values kernels

// A = w (Eq. 1) into shared memory, NoData -> marker (D9); returns
// sum w over data cells (integer weights: the u32 overflow check, D10)
template <class T, int WK, class S>
__device__ __forceinline__ unsigned long long init_values_v(S& s, const void* wp, const Geom& g, int64_t y0,
                                                            int64_t x0, int h, int w, uint32_t* status) {
  using WB = typename S::WB;
  const int lane = lane_id();
  unsigned long long wsum = 0;
  bool bad = false;
  const bool vec = WK != 0 && w == WB::BC && ((x0 & 3) == 0) && ((g.W & 3) == 0) &&
                   ((reinterpret_cast<uintptr_t>(wp) & 15) == 0);
  const uint32_t* W32 = static_cast<const uint32_t*>(wp);
  for (int q = lane; q < h * (WB::BC / 4); q += 32) {
    const int ly = q >> 3, lx = (q & 7) * 4;
    const uint32_t dw = *reinterpret_cast<const uint32_t*>(&s.dirh[WB::hidx(ly, lx)]);
    const int64_t gi = (y0 + ly) * g.W + x0 + lx;
    uint32_t u[4] = {1u, 1u, 1u, 1u};
    if (WK != 0) {
      if (vec) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(W32 + gi));
        u[0] = v.x; u[1] = v.y; u[2] = v.z; u[3] = v.w;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (lx + j < w) u[j] = __ldg(W32 + gi + j);
      }
    }
    alignas(16) T v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int code = (dw >> (8 * j)) & 0xFF;
      const bool data = code < kOut;
      if constexpr (WK == 0) {
        v[j] = (T)1;
      } else if constexpr (WK == 1) {
        v[j] = (T)u[j];
        if (data) wsum += u[j];
      } else {
        const float f = __uint_as_float(u[j]);
        if (data && !weight_ok<WK>(f)) bad = true;
        v[j] = (T)f;
      }
      if (code == kNoData) v[j] = AccT<T>::marker();
    }
    if constexpr (sizeof(T) == 4) {
      *reinterpret_cast<uint4*>(&s.a[4 * q]) = *reinterpret_cast<const uint4*>(v);
    } else {
      reinterpret_cast<uint4*>(&s.a[4 * q])[0] = *reinterpret_cast<const uint4*>(&v[0]);
      reinterpret_cast<uint4*>(&s.a[4 * q])[1] = *reinterpret_cast<const uint4*>(&v[2]);
    }
  }
  if (bad) atomicOr(status, ST_BADWEIGHT);
  return wsum;
}

// In-block donor counts (one byte per cell) by an 8-neighbour SWAR gather --
// 4 cells per 32-bit word, no atomics (Alg. 1's first loop) --
// plus the successor words (as build_masks) and the sources queue.  Returns
// this lane's data-cell count; nsrc = number of sources (warp total).
template <bool SUCC, class S>
__device__ __forceinline__ int build_counts_v(S& s, uint32_t& nsrc, int h, int w) {
  using WB = typename S::WB;
  constexpr int R = S::RR;
  constexpr int NQ = WB::BN / 128;
  constexpr int RW = WB::HS / 4;
  const int lane = lane_id();
  const uint32_t* D = reinterpret_cast<const uint32_t*>(s.dirh);
  uint32_t* C = reinterpret_cast<uint32_t*>(s.cnt);
  int ndata = 0;
  uint32_t srcbits = 0, ndbits = 0;
  auto eq7 = [](uint32_t n, uint32_t c) {  // bit 7 of byte j set iff byte j of n equals c (see donor_masks)
    const uint32_t y = ((n ^ c) & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;
    return (~(y | n) & 0x80808080u) >> 7;
  };
#pragma unroll 2
  for (int k = 0; k < NQ; ++k) {
    const int q = k * 32 + lane;
    const int ly = q >> 3, lx0 = (q & 7) * 4;
    const int hw = WB::hidx(ly, lx0) >> 2;
    const uint32_t u0 = D[hw - RW - 1], u1 = D[hw - RW], u2 = D[hw - RW + 1];
    const uint32_t c0 = D[hw - 1], c1 = D[hw], c2 = D[hw + 1];
    const uint32_t d0 = D[hw + RW - 1], d1 = D[hw + RW], d2 = D[hw + RW + 1];
    // count = number of neighbours n whose code is opp(direction to n)
    uint32_t cnt = eq7(u1, 0x05050505u) + eq7(__funnelshift_r(u1, u2, 8), 0x06060606u) +
                   eq7(__funnelshift_r(c1, c2, 8), 0x07070707u) + eq7(__funnelshift_r(d1, d2, 8), 0x08080808u) +
                   eq7(d1, 0x01010101u) + eq7(__funnelshift_r(d0, d1, 24), 0x02020202u) +
                   eq7(__funnelshift_r(c0, c1, 24), 0x03030303u) + eq7(__funnelshift_r(u0, u1, 24), 0x04040404u);
    const uint32_t nd = __vcmpgeu4(c1, 0xFEFEFEFEu);  // NoData / outside the block: not a cell
    const uint32_t inb = ly >= h ? 0u : lx0 + 4 <= w ? 0xFFFFFFFFu : lx0 >= w ? 0u : (0xFFFFFFFFu >> (8 * (lx0 + 4 - w)));
    // in-block NoData with donors: stop them below (with fused D8 their
    // successor words say so already: d8_put, the | 16 of an outlet code)
    const uint32_t sink = SUCC ? (nd & inb & ~__vcmpeq4(cnt, 0u)) : 0u;
    ndbits |= (sink ? 1u : 0u) << k;
    cnt &= ~nd;
    C[q] = cnt;
    ndata += 4 - (__popc(nd) >> 3);
    const uint32_t src4 = __vcmpeq4(cnt, 0u) & ~nd & 0x80808080u;
    srcbits |= (((src4 >> 7) & 1u) | ((src4 >> 14) & 2u) | ((src4 >> 21) & 4u) | ((src4 >> 28) & 8u)) << (4 * k);
    if constexpr (!SUCC) continue;
    uint32_t sbw;
    if (h == WB::BR && w == WB::BC) {
      // full block: the codes plus SB_EXIT on the border (see build_masks)
      const uint32_t nib = code_nibbles(c1);
      sbw = sb_word(c1, nib, border_exits<WB::BR>(nib, ly, lx0));
    } else {
      sbw = 0u;
      const uint32_t fr = forb_row(ly, h);
#pragma unroll
      for (int j = 0; j < 4; ++j) sbw |= succ_byte((c1 >> (8 * j)) & 0xFF, fr | forb_col(lx0 + j, w)) << (8 * j);
    }
    reinterpret_cast<uint32_t*>(s.sb)[q] = sbw;
  }
  if (SUCC && __any_sync(kFull, ndbits != 0u)) {
    // donors of in-block NoData cells: their flow is dropped (STOP, D8)
    __syncwarp();
#pragma unroll 1
    for (int k = 0; k < NQ; ++k) {
      if (!((ndbits >> k) & 1u)) continue;
      const int q = k * 32 + lane;
      const int hw = WB::hidx(q >> 3, (q & 7) * 4) >> 2;
      const uint32_t pw = donor_masks<R>(D, hw);
      const int ly = q >> 3, lx0 = (q & 7) * 4;
      const uint32_t inb = ly >= h ? 0u : lx0 + 4 <= w ? 0xFFFFFFFFu : lx0 >= w ? 0u : (0xFFFFFFFFu >> (8 * (lx0 + 4 - w)));
      const uint32_t nd = __vcmpgeu4(D[hw], 0xFEFEFEFEu) & inb;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (!((nd >> (8 * j)) & 1u)) continue;
        uint32_t mm = (pw >> (8 * j)) & 0xFFu;
        while (mm) {
          const int kk = __ffs(mm);
          mm &= mm - 1;
          s.sb[4 * q + j + WB::offA(kk)] = (uint8_t)(SB_STOP | SB_DROP);
        }
      }
    }
  }
  const int c = __popc(srcbits);
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += v;
  }
  nsrc = (uint32_t)__shfl_sync(kFull, incl, 31);
  int pos = incl - c;
  while (srcbits) {
    const int bpos = __ffs(srcbits) - 1;
    srcbits &= srcbits - 1;
    FA_CHECK(pos < WB::BN);
    s.src[pos++] = (uint16_t)(4 * ((bpos >> 2) * 32 + lane) + (bpos & 3));
  }
  return ndata;
}

// Alg. 1, "the last donor continues" with conflict-free pushes (see above).
// Returns the number of cells retired (sources + cells whose count reached
// zero), warp total.
template <class S>
__device__ __forceinline__ uint32_t kahn_push(S& s, uint32_t nsrc) {
  using T = typename S::VT;
  using WB = typename S::WB;
  const int lane = lane_id();
  const unsigned lt = (1u << lane) - 1u;
  uint32_t head = 0, done = 0;
  int cur = -1;
  T a = (T)0;
  for (;;) {
    __syncwarp();
    const unsigned idle = __ballot_sync(kFull, cur < 0);
    if (idle == kFull && head >= nsrc) break;
    if (cur < 0) {
      const uint32_t r = head + (uint32_t)__popc(idle & lt);
      if (r < nsrc) {
        cur = s.src[r];
        a = s.a[cur];  // a source: A = w, final
        ++done;
      }
    }
    head = min(head + (uint32_t)__popc(idle), nsrc);
    const uint32_t sbv = cur >= 0 ? (uint32_t)s.sb[cur] : SB_STOP;
    const bool go = sb_go(sbv);
    if (!go) cur = -1;  // NoFlow, NoData target or a block exit: A(cur) is final and stored
    // one pusher per target cell and iteration: every pusher writes its lane
    // into the target's claim byte, the lane read back pushes, the others retry
    const uint32_t t = go ? WB::target((uint32_t)cur, sbv) : 0u;
    FA_CHECK(t < (uint32_t)WB::BN);
    if (go) s.claim[t] = (uint8_t)lane;
    __syncwarp();
    if (go && s.claim[t] == (uint8_t)lane) {
      // "A(n) <- A(n) + A(c)", "decrement D(n)" (Alg. 1)
      const T at = s.a[t] + a;
      s.a[t] = at;
      const uint32_t c = (uint32_t)s.cnt[t] - 1u;
      s.cnt[t] = (uint8_t)c;
      if (c == 0u) {  // the last donor: A(n) is final, continue from n
        cur = (int)t;
        a = at;
        ++done;
      } else {
        cur = -1;
      }
    }
  }
  __syncwarp();
  return __reduce_add_sync(kFull, done);
}

// the block's values to the output (16-byte rows when aligned)
template <class T, class S>
__device__ __forceinline__ void write_values(const S& s, T* out, const Geom& g, int64_t y0, int64_t x0, int h,
                                             int w) {
  using WB = typename S::WB;
  const int lane = lane_id();
  const bool vec = w == WB::BC && ((x0 & 3) == 0) && ((g.W & 3) == 0) &&
                   ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  if (vec) {
    for (int q = lane; q < h * (WB::BC / 4); q += 32) {
      const int ly = q >> 3, lx = (q & 7) * 4;
      T* dst = out + (y0 + ly) * g.W + x0 + lx;
      if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(&s.a[4 * q]);
      } else {
        reinterpret_cast<uint4*>(dst)[0] = reinterpret_cast<const uint4*>(&s.a[4 * q])[0];
        reinterpret_cast<uint4*>(dst)[1] = reinterpret_cast<const uint4*>(&s.a[4 * q])[1];
      }
    }
  } else {
    for (int i = lane; i < h * WB::BC; i += 32) {
      const int ly = i >> 5, lx = i & 31;
      if (lx < w) out[(y0 + ly) * g.W + x0 + lx] = s.a[i];
    }
  }
}

template <class T, int R, int WK, bool FROM_DEM = false>
__global__ void __launch_bounds__(32 * kNWV) k_pass1v(PassArgs<T, WK> P) {
  using WB = WBT<R>;
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  VSmem<T, R>& s = reinterpret_cast<VSmem<T, R>*>(smem)[warp];
  const Geom& g = P.g;
  const int64_t b = P.b_begin + (int64_t)blockIdx.x * kNWV + warp;
  if (b >= P.b_end) return;
  const int lane = lane_id();
  int64_t y0, x0;
  int h, w;
  g.block_box(b, y0, x0, h, w);
  if (h <= 0 || w <= 0) {
    for (int p = lane; p < WB::PB; p += 32) P.slot_root[b * WB::PB + p] = kNone;
    return;
  }
  init_smem(s);
  if constexpr (FROM_DEM) {
    // N1: H1 fused -- the z window is staged in the values' room, the codes
    // and successor words come from the D8 stencil, the ring's D8 marks the
    // entries; the codes also go to the output for the finalize
    stage_z(s, P, y0, x0, h, w);
    __syncwarp();
    d8_block(s, h, w);
    ring_entries(s, P, y0, h, w);
    __syncwarp();
    if (P.dirs_out) write_dirs(s, P.dirs_out, g, y0, x0, h, w);
  } else {
    __syncwarp();
    load_dirs(s, P.dirs_in, P.dirs_up, P.dirs_dn, g, y0, x0, h, w, true, true, P.status);
  }
  __syncwarp();
  uint32_t nsrc;
  const int ndata = build_counts_v<!FROM_DEM>(s, nsrc, h, w);
  __syncwarp();  // the z window (fused D8) is dead: A = w takes its place
  unsigned long long wsum = init_values_v<T, WK>(s, P.w, g, y0, x0, h, w, P.status);
  const uint32_t popped = kahn_push(s, nsrc);
  const int tot_data = __reduce_add_sync(kFull, ndata);
  if (lane == 0 && (int)popped != tot_data) atomicOr(P.status, ST_CYCLE);  // a cell never became ready
  if (!std::is_same<T, double>::value && P.wsum) {
    if (WK == 0) wsum = lane == 0 ? (unsigned long long)tot_data : 0;
    for (int o = 16; o; o >>= 1) wsum += __shfl_xor_sync(kFull, wsum, o);
    if (lane == 0 && wsum) atomicAdd(P.wsum, wsum);
  }
  if (P.retain) write_values(s, P.acc, g, y0, x0, h, w);  // RETAIN: A_B into the output
  block_records<T, R, VSmem<T, R>, WK>(s, P, b, y0, x0, h, w);
}

// EVICT pass 2: the block again with w + x, x = the external
// inbound flow of each entry slot (D11, D12), values on chip
template <class T, int R, int WK>
__global__ void __launch_bounds__(32 * kNWV) k_pass2v(PassArgs<T, WK> P) {
  using WB = WBT<R>;
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  VSmem<T, R>& s = reinterpret_cast<VSmem<T, R>*>(smem)[warp];
  const Geom& g = P.g;
  const int64_t b = P.b_begin + (int64_t)blockIdx.x * kNWV + warp;
  if (b >= P.b_end) return;
  const int lane = lane_id();
  int64_t y0, x0;
  int h, w;
  g.block_box(b, y0, x0, h, w);
  if (h <= 0 || w <= 0) return;
  init_smem(s);
  __syncwarp();
  load_dirs(s, P.dirs_in, P.dirs_up, P.dirs_dn, g, y0, x0, h, w, false, false, P.status);
  __syncwarp();
  uint32_t nsrc;
  const int ndata = build_counts_v<true>(s, nsrc, h, w);
  init_values_v<T, WK>(s, P.w, g, y0, x0, h, w, P.status);
  __syncwarp();
  const int np = bperim_count(h, w);
  for (int p = lane; p < np; p += 32) {  // inject x at the block perimeter (distinct cells per lane)
    int px, py;
    bperim_xy(p, h, w, px, py);
    if (s.dirh[WB::hidx(py, px)] == kNoData) continue;
    s.a[py * WB::BC + px] += P.x_slot[b * WB::PB + p];
  }
  const uint32_t popped = kahn_push(s, nsrc);
  const int tot_data = __reduce_add_sync(kFull, ndata);
  if (lane == 0 && (int)popped != tot_data) atomicOr(P.status, ST_CYCLE);
  write_values(s, P.acc, g, y0, x0, h, w);
}

// ---------------------------------------------------------------- RETAIN finalize
// "add A' to every cell in its downstream flow path" (Alg. 3): acc
// already holds the block-local accumulation written by pass 1.  A warp owns
// KB consecutive blocks (1 by default): it stages their codes in shared memory, compacts
// the entry slots with a non-zero offset x (x = external inbound flow, D11)
// into a work list, and its lanes walk those entries' in-block paths, adding
// x to every cell up to the block exit or the NoFlow terminal (flow into
// NoData is dropped, D8) with fire-and-forget global atomics; a lane whose
// walk ends takes the next entry.  A = A_B + the offsets whose path passes
// the cell (linearity, D12).
// codes of a staged block (row stride 32) -> successor bytes in place
// (sb_word; the finalize's walks).  Bytes > 8 other than NoData (bad codes,
// already rejected by pass 1) read as NoData, so a walk can never leave the
// block's cells.
template <int R>
__device__ __forceinline__ void succ_bytes_inplace(uint8_t* d, int h, int w) {
  uint32_t* D = reinterpret_cast<uint32_t*>(d);
  for (int q = lane_id(); q < h * 8; q += 32) {
    const int ly = q >> 3, lx0 = (q & 7) * 4;
    const uint32_t c1 = D[q] | __vcmpgtu4(D[q], 0x08080808u);
    uint32_t sbw;
    if (h == R && w == 32) {
      const uint32_t nib = code_nibbles(c1);
      sbw = sb_word(c1, nib, border_exits<R>(nib, ly, lx0));
    } else {
      sbw = 0u;
      const uint32_t fr = forb_row(ly, h);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        sbw |= (lx0 + j < w ? succ_byte((c1 >> (8 * j)) & 0xFF, fr | forb_col(lx0 + j, w)) : (uint32_t)kNoData)
               << (8 * j);
    }
    D[q] = sbw;
  }
  __syncwarp();
}

template <class T, int R, int KB>
struct __align__(16) FSmem {
  using WB = WBT<R>;
  uint8_t d[KB][WB::BN];                 // codes of the KB blocks (row stride 32)
  uint16_t item[KB * WB::PB];            // work list: (block-in-group << 8) | slot
};

template <class T, int R, int KB, bool ABS = false, bool FULL = false>
__global__ void __launch_bounds__(128) k_finalize(Geom g, const T* __restrict__ x_slot, const uint8_t* __restrict__ dirs,
                                                  T* acc, const float* __restrict__ alpha, int64_t bbeg, int64_t bend) {
  using WB = WBT<R>;
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  FSmem<T, R, KB>& s = reinterpret_cast<FSmem<T, R, KB>*>(smem)[warp];
  const int64_t b0 = bbeg + ((int64_t)blockIdx.x * (blockDim.x >> 5) + warp) * KB;
  if (b0 >= bend) return;
  const int lane = lane_id();
  const unsigned lt = (1u << lane) - 1u;
  int64_t y0s[KB], x0s[KB];
  int hs[KB], ws[KB];
  int n = 0;  // work items (warp-uniform)
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    const int64_t b = b0 + k;
    hs[k] = ws[k] = 0;
    y0s[k] = x0s[k] = 0;
    if (b < bend) g.block_box(b, y0s[k], x0s[k], hs[k], ws[k]);
    if (FULL && hs[k] > 0 && ws[k] > 0) {  // whole blocks: the shape as constants
      hs[k] = R;
      ws[k] = 32;
    }
    // the block's work list first: a block no offset reaches (NoData, ridges)
    // skips the prefetch and the code staging
    const int n0 = n;
    const int np = bperim_count(hs[k], ws[k]);
    for (int p0 = 0; p0 < WB::PB; p0 += 32) {
      const int p = p0 + lane;
      const bool act = p < np && x_slot[b * WB::PB + p] != (T)0;
      const unsigned m = __ballot_sync(kFull, act);
      if (act) s.item[n + __popc(m & lt)] = (uint16_t)((k << 8) | p);
      n += __popc(m);
    }
    if (n == n0 || hs[k] <= 0 || ws[k] <= 0) continue;
#if FA_FIN_PREFETCH
    // pull the block's output rows into L2 before the walks' reductions
    // reach them: a reduction on a line that is not in L2 waits for its DRAM
    // fill inside the L2 atomic unit, while prefetches stream (the rows were
    // written by pass 1 long ago and are cold)
    for (int i = lane; i < hs[k] * FA_FIN_PREFETCH; i += 32) {
      const int ly = i / FA_FIN_PREFETCH, part = i - ly * FA_FIN_PREFETCH;
      const T* row = acc + (y0s[k] + ly) * g.W + x0s[k];
      const char* ptr = reinterpret_cast<const char*>(row) + part * (WB::BC * (int)sizeof(T) / FA_FIN_PREFETCH);
      if (part * (WB::BC / FA_FIN_PREFETCH) < ws[k]) asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
    }
#endif
    // codes: 16-byte rows when aligned
    const int h = hs[k], w = ws[k];
    const bool vec = w == WB::BC && ((x0s[k] & 15) == 0) && ((g.W & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(dirs) & 15) == 0);
    if (vec) {
      for (int q = lane; q < h * 2; q += 32) {
        const int ly = q >> 1, lx = (q & 1) * 16;
        *reinterpret_cast<uint4*>(&s.d[k][ly * WB::BC + lx]) =
            __ldg(reinterpret_cast<const uint4*>(dirs + (y0s[k] + ly) * g.W + x0s[k] + lx));
      }
    } else {
      for (int i = lane; i < h * WB::BC; i += 32) {
        const int ly = i >> 5, lx = i & 31;
        if (lx < w) s.d[k][i] = dirs[(y0s[k] + ly) * g.W + x0s[k] + lx];
      }
    }
    __syncwarp();
    succ_bytes_inplace<R>(s.d[k], h, w);
  }
  __syncwarp();
  // walks over block cell indices c = 32*ly + lx: a step is one byte load,
  // one reduction, one compare and one add (successor bytes, see sb_word)
  const uint32_t wm = (uint32_t)g.W - 32u;
  int head = 0, k = -1;
  uint32_t c = 0;
  T x = (T)0;
  T* rowp = nullptr;  // acc + y0 * W + x0 of the walk's block
  const float* arow = nullptr;  // absorption: alpha + y0 * W + x0
  for (;;) {
    const unsigned idle = __ballot_sync(kFull, k < 0);
    if (idle == kFull && head >= n) break;
    if (k < 0) {
      const int r = head + __popc(idle & lt);
      if (r < n) {
        const int it = s.item[r];
        k = it >> 8;
        const int p = it & 0xFF;
        int kk = 0;
#pragma unroll
        for (int j = 1; j < KB; ++j) kk = k == j ? j : kk;
        int h = hs[0], w = ws[0];
        int64_t yy = y0s[0], xx = x0s[0];
#pragma unroll
        for (int j = 1; j < KB; ++j)
          if (kk == j) { h = hs[j]; w = ws[j]; yy = y0s[j]; xx = x0s[j]; }
        x = x_slot[(b0 + k) * WB::PB + p];
        rowp = acc + yy * g.W + xx;
        if (ABS) arow = alpha + yy * g.W + xx;
        int cx, cy;
        bperim_xy(p, h, w, cx, cy);
        c = (uint32_t)(cy * WB::BC + cx);
      }
    }
    head += __popc(idle);
    if (k < 0) continue;
    // FA_FIN_STEPS path steps per refill round (the refill bookkeeping is
    // paid once per round)
#pragma unroll
    for (int u = 0; u < FA_FIN_STEPS; ++u) {
      FA_CHECK(c < (uint32_t)WB::BN);
      const uint32_t sb = s.d[k][c];
      // a walk that reaches in-block NoData stops there: the flow is dropped (D8)
      if (sb == kNoData) { k = -1; break; }
      const uint32_t off = cell_off(c, wm);
      g_add(elt(rowp, off), x);
      if (!sb_go(sb)) { k = -1; break; }  // terminal or block exit
      if (ABS) x *= (T)__ldg(arow + off);  // the cell passes on alpha of it
      c = WB::target(c, sb);
    }
  }
}

// every non-empty block of the geometry is a whole R x 32 block (the raster,
// strip and tile sizes are multiples of the block shape; cfg0-4): kernels
// specialised for it have the block shape as constants
static bool whole_blocks(const Geom& g, int R) {
  return R == 32 && g.H % R == 0 && g.W % 32 == 0 && (g.TH % R == 0 || g.TH >= g.H) &&
         (g.TW % 32 == 0 || g.TW >= g.W);
}

template <class T, int R, int KB>
cudaError_t launch_finalize_k(const Geom& g, const T* x_slot, const uint8_t* dirs, T* acc, cudaStream_t st,
                              int64_t bbeg, int64_t bend) {
  constexpr int NWC = FA_FIN_NW;  // warps per CTA
  // At least 6 KB of shared memory per warp: at most 36 warps per SM, which
  // keeps the acc rows the walks touch in L2 (measured on cfg3: 3.82 ms vs
  // 3.92 ms at full occupancy).
  size_t sm = sizeof(FSmem<T, R, KB>) * NWC;
  sm = sm < FA_FIN_SMEM_FLOOR * NWC ? FA_FIN_SMEM_FLOOR * NWC : sm;
  auto k = whole_blocks(g, R) ? k_finalize<T, R, KB, false, R == 32> : k_finalize<T, R, KB>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const int64_t groups = (bend - bbeg + KB - 1) / KB;
  k<<<(unsigned)((groups + NWC - 1) / NWC), 32 * NWC, sm, st>>>(g, x_slot, dirs, acc, nullptr, bbeg, bend);
  return cudaGetLastError();
}

// one block per warp (2 or 4 measured slower on cfg3)
template <class T, int R>
cudaError_t launch_finalize_r(const Geom& g, const T* x_slot, const uint8_t* dirs, T* acc, cudaStream_t st,
                              int64_t bbeg, int64_t bend) {
  return launch_finalize_k<T, R, 1>(g, x_slot, dirs, acc, st, bbeg, bend);
}

// CTAs of a pass-1 launch over n blocks: nw warps per CTA, FA_P1_KPW blocks per warp
static unsigned p1_grid(int64_t n, int nw) {
  const int64_t per = (int64_t)nw * FA_P1_KPW;
  return (unsigned)((n + per - 1) / per);
}

// absorption (f64, 32x32 blocks): pass 1 and the finalize with alpha
cudaError_t launch_pass1_absorb(const PassArgs<double, 0>* a0, const PassArgs<double, 2>* a2, bool from_dem,
                                cudaStream_t st) {
  auto go = [&](auto k, const auto& a) {
    const size_t sm = (from_dem ? sizeof(WSmem<double, 32, true>) : sizeof(WSmem<double, 32, false>)) * (size_t)a.g.nw;
    const unsigned grid = p1_grid(a.b_end - a.b_begin, a.g.nw);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<grid, 32 * a.g.nw, sm, st>>>(a);
  };
  if (a0) {
    if (a0->g.br != 32 || a0->g.bc != 32) return cudaErrorInvalidValue;
    if (from_dem) go(k_pass1<double, 32, 0, true, true>, *a0);
    else if (whole_blocks(a0->g, 32)) go(k_pass1<double, 32, 0, false, true, true>, *a0);
    else go(k_pass1<double, 32, 0, false, true>, *a0);
  } else {
    if (a2->g.br != 32 || a2->g.bc != 32) return cudaErrorInvalidValue;
    if (from_dem) go(k_pass1<double, 32, 2, true, true>, *a2);
    else if (whole_blocks(a2->g, 32)) go(k_pass1<double, 32, 2, false, true, true>, *a2);
    else go(k_pass1<double, 32, 2, false, true>, *a2);
  }
  return cudaGetLastError();
}

cudaError_t launch_retain_absorb(const Geom& g, const double* x_slot, const uint8_t* dirs, double* acc,
                                 const float* alpha, cudaStream_t st) {
  if (g.br != 32 || g.bc != 32) return cudaErrorInvalidValue;
  constexpr int NWC = 4;
  size_t sm = sizeof(FSmem<double, 32, 1>) * NWC;
  sm = sm < 24576 ? 24576 : sm;
  auto k = whole_blocks(g, 32) ? k_finalize<double, 32, 1, true, true> : k_finalize<double, 32, 1, true>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k<<<(unsigned)((g.nblocks + NWC - 1) / NWC), 32 * NWC, sm, st>>>(g, x_slot, dirs, acc, alpha, 0, g.nblocks);
  return cudaGetLastError();
}

// bend < 0: every block
template <class T>
cudaError_t launch_retain(const Geom& g, const T* x_slot, const uint8_t* dirs, T* acc, cudaStream_t st,
                          int64_t bbeg, int64_t bend) {
  if (g.bc != 32) return cudaErrorInvalidValue;
  if (bend < 0) bend = g.nblocks;
  if (bend <= bbeg) return cudaSuccess;
  if (g.br == 32) return launch_finalize_r<T, 32>(g, x_slot, dirs, acc, st, bbeg, bend);
  if (g.br == 16) return launch_finalize_r<T, 16>(g, x_slot, dirs, acc, st, bbeg, bend);
  if (g.br == 64) return launch_finalize_r<T, 64>(g, x_slot, dirs, acc, st, bbeg, bend);
  return cudaErrorInvalidValue;
}
template cudaError_t launch_retain<uint32_t>(const Geom&, const uint32_t*, const uint8_t*, uint32_t*, cudaStream_t,
                                             int64_t, int64_t);
template cudaError_t launch_retain<unsigned long long>(const Geom&, const unsigned long long*, const uint8_t*,
                                                       unsigned long long*, cudaStream_t, int64_t, int64_t);
template cudaError_t launch_retain<double>(const Geom&, const double*, const uint8_t*, double*, cudaStream_t, int64_t,
                                           int64_t);

// ---------------------------------------------------------------- launchers
// pass 1: the block's values on chip (k_pass1v) or in the output raster
// (k_pass1), FA_OPT_VALUES; either with D8 fused (FA_OPT_D8 = FA_D8_FUSED:
// the z window staged in shared memory) or from the D8 raster
template <class T, int R, int WK>
cudaError_t launch_pass1_r(const PassArgs<T, WK>& a, bool from_dem, cudaStream_t st) {
  if (a.vsmem) {
    const size_t sm = sizeof(VSmem<T, R>) * (size_t)kNWV;
    const unsigned grid = (unsigned)((a.b_end - a.b_begin + kNWV - 1) / kNWV);
    auto k = from_dem ? k_pass1v<T, R, WK, true> : k_pass1v<T, R, WK, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<grid, 32 * kNWV, sm, st>>>(a);
  } else if (from_dem) {
    const size_t sm = sizeof(WSmem<T, R, true>) * (size_t)a.g.nw;
    const unsigned grid = p1_grid(a.b_end - a.b_begin, a.g.nw);
    auto k = k_pass1<T, R, WK, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<grid, 32 * a.g.nw, sm, st>>>(a);
  } else {
    const size_t sm = sizeof(WSmem<T, R, false>) * (size_t)a.g.nw;
    const unsigned grid = p1_grid(a.b_end - a.b_begin, a.g.nw);
    auto k = whole_blocks(a.g, R) ? k_pass1<T, R, WK, false, false, R == 32> : k_pass1<T, R, WK, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<grid, 32 * a.g.nw, sm, st>>>(a);
  }
  return cudaGetLastError();
}

template <class T, int R, int WK>
cudaError_t launch_pass2_r(const PassArgs<T, WK>& a, cudaStream_t st) {
  if (!a.vsmem) {
    const size_t sm = sizeof(WSmem<T, R, false>) * (size_t)a.g.nw;
    const unsigned grid = (unsigned)((a.b_end - a.b_begin + a.g.nw - 1) / a.g.nw);
    auto k = k_pass2<T, R, WK>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<grid, 32 * a.g.nw, sm, st>>>(a);
    return cudaGetLastError();
  }
  const size_t sm = sizeof(VSmem<T, R>) * (size_t)kNWV;
  const unsigned grid = (unsigned)((a.b_end - a.b_begin + kNWV - 1) / kNWV);
  auto k = k_pass2v<T, R, WK>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k<<<grid, 32 * kNWV, sm, st>>>(a);
  return cudaGetLastError();
}

template <class T, int WK>
cudaError_t launch_pass1(const PassArgs<T, WK>& a, bool from_dem, cudaStream_t st) {
  if (a.g.bc != 32 || a.g.nw < 1 || a.g.nw > 4) return cudaErrorInvalidValue;
  if (a.g.br == 32) return launch_pass1_r<T, 32, WK>(a, from_dem, st);
  if (a.g.br == 16) return launch_pass1_r<T, 16, WK>(a, from_dem, st);
  if (a.g.br == 64) return launch_pass1_r<T, 64, WK>(a, from_dem, st);
  return cudaErrorInvalidValue;
}

template <class T, int WK>
cudaError_t launch_pass2(const PassArgs<T, WK>& a, cudaStream_t st) {
  if (a.g.bc != 32 || a.g.nw < 1 || a.g.nw > 4) return cudaErrorInvalidValue;
  if (a.g.br == 32) return launch_pass2_r<T, 32, WK>(a, st);
  if (a.g.br == 16) return launch_pass2_r<T, 16, WK>(a, st);
  if (a.g.br == 64) return launch_pass2_r<T, 64, WK>(a, st);
  return cudaErrorInvalidValue;
}

#define FA_INST(T, WK)                                                              \
  template cudaError_t launch_pass1<T, WK>(const PassArgs<T, WK>&, bool, cudaStream_t); \
  template cudaError_t launch_pass2<T, WK>(const PassArgs<T, WK>&, cudaStream_t);
FA_INST(uint32_t, 0)
FA_INST(uint32_t, 1)
FA_INST(unsigned long long, 0)
FA_INST(unsigned long long, 1)
FA_INST(double, 0)
FA_INST(double, 2)
#undef FA_INST

}  // namespace fa
