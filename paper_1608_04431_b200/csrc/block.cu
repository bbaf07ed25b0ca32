// block.cu -- CTA-resident block kernels (SURVEY N1 "SMEM-resident fused tile
// kernel"): each CTA owns a BR x BC block and runs the paper's single-tile
// algorithm on it entirely in shared memory.
//
//   pass 1 (k_pass1): [H1 D8 from the DEM + 1-cell halo] -> [H2 in-block donor
//     masks by an 8-neighbour gather, no atomics] -> [H3 in-block accumulation,
//     Alg. 1 P:L127-176] -> [H4 block perimeter records: one node per block exit
//     cell with its block-local accumulation, and for every perimeter cell the
//     exit its in-block path reaches, Alg. 2 P:L178-204].
//   pass 2 (k_pass2): [H6 offset propagation, EVICT P:L255-262]: rerun H2-H3 with
//     w + x at the block perimeter cells (x = external inbound flow, D11/D12).
//
// H3 scheduling (differs from the paper's FIFO): walks.  The
// block's sources (data cells without in-block donors) are compacted into a
// shared queue.  A lane takes a source and walks downstream, adding its value
// into the next cell and continuing while it is that cell's only pending
// donor -- cells with exactly one donor need no atomic.  At a junction the
// walk clears its bit in the target's pending-donor mask (one shared
// atomicAnd on a packed word); only the last arrival gathers the donors'
// values (fixed donor order) and continues.  A lane whose walk ends takes the
// next source at once, so lanes stay busy while a few long rivers are walked.
//
// Why small blocks (default 32 x 32, one warp): a block's walks finish no
// sooner than its longest in-block flow path, so throughput = cells in flight
// per SM / block latency.  Shared memory bounds the cells in flight (~14 KB
// per 32x32 f64 block -> 16 blocks per SM); smaller blocks shorten the
// critical path (ncu on 64x64 blocks: 25 % occupancy, issue 35 %, stalls on
// global loads and on the end-of-walk barrier).
//
// Shared-memory layout: directions are stored with a 1-cell halo ring, row
// stride HS = BC + 8 with the block interior at column 4 (4-byte aligned rows
// for SWAR); ring cells hold 254 (outside the block) or 255 (NoData /
// off-grid), so walks need no bounds tests.  Masks and values use stride BC.
#include "fa_internal.cuh"

namespace fa {

constexpr uint8_t kOut = 254;  // ring cell: outside the block, data

// Optional per-phase cycle accounting (profiling build only, -DFA_PHASE_CLOCKS):
// thread 0 of every CTA adds the cycles each phase took to g_phase[i].
#ifdef FA_PHASE_CLOCKS
__device__ unsigned long long g_phase[16];
#define PH_T0 long long _ph_t = clock64()
#define PH_MARK(i)                                                          \
  do {                                                                      \
    if (threadIdx.x == 0) {                                                 \
      const long long _n = clock64();                                       \
      atomicAdd(&g_phase[i], (unsigned long long)(_n - _ph_t));             \
      _ph_t = _n;                                                           \
    }                                                                       \
  } while (0)
}  // namespace fa
extern "C" __attribute__((visibility("default"))) int fa_debug_phase_clocks(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, fa::g_phase, sizeof(fa::g_phase)) != cudaSuccess) return 1;
  if (reset) {
    static const unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(fa::g_phase, z, sizeof(z));
  }
  return 0;
}
namespace fa {
#else
#define PH_T0 (void)0
#define PH_MARK(i) (void)0
#endif

// packed signed 8-bit offsets of direction codes 1..8 for a row stride S
__host__ __device__ constexpr uint64_t pack_offsets(int S) {
  uint64_t t = 0;
  for (int k = 1; k <= 8; ++k)
    t |= (uint64_t)(uint8_t)(int8_t)(dir_dy(k) * S + dir_dx(k)) << (8 * (k - 1));
  return t;
}

template <int BR_, int BC_, int NW_>
struct Cfg {
  static constexpr int BR = BR_, BC = BC_, NW = NW_;
  static constexpr int NT = 32 * NW;
  static constexpr int BN = BR * BC;
  static constexpr int PB = 2 * (BR + BC) - 4;
  static constexpr int HS = BC + 8;               // halo'd row stride (interior at col 4)
  static constexpr int HN = (BR + 2) * HS;
  static constexpr int ZS = BC + 2;               // staged elevations stride
  static constexpr int ZN = (BR + 2) * ZS;
  static constexpr uint64_t OFFH = pack_offsets(HS);
  static constexpr uint64_t OFFA = pack_offsets(BC);
  static_assert(BC % 4 == 0 && BN % (4 * NT) == 0, "block shape");
  static_assert(HS <= 120, "int8 offsets");
  __device__ static __forceinline__ int offH(int d) { return (int)(int8_t)(OFFH >> (8 * (d - 1))); }
  __device__ static __forceinline__ int offA(int d) { return (int)(int8_t)(OFFA >> (8 * (d - 1))); }
  __device__ static __forceinline__ int hidx(int ly, int lx) { return (ly + 1) * HS + lx + 4; }
  __device__ static __forceinline__ int a2h(int i) { return hidx(i / BC, i % BC); }
};

template <class C>
struct __align__(16) Smem {
  uint8_t dirh[C::HN];
  uint32_t msk4[C::BN / 4];  // donor masks, one byte per cell
  uint32_t pend[C::BN / 4];  // pending-donor masks (atomicAnd)
  uint16_t src[C::BN];       // source queue (A index)
  uint32_t slot_nid[C::PB];
  uint32_t nsrc, qhead, cnt_exit, base, processed, ndata;
  __device__ __forceinline__ uint8_t msk(int i) const { return reinterpret_cast<const uint8_t*>(msk4)[i]; }
};

template <class C, class T>
struct SmemSize {
  static constexpr size_t a_bytes = sizeof(T) * C::BN;
  static constexpr size_t z_bytes = sizeof(float) * C::ZN;
  static constexpr size_t region = ((a_bytes > z_bytes ? a_bytes : z_bytes) + 15) / 16 * 16;
  static constexpr size_t total = region + sizeof(Smem<C>);
};

template <int WK>
__device__ __forceinline__ bool weight_ok(float v) {
  return WK != 2 || (isfinite(v) && v >= 0.0f);  // D21
}

template <class T, int WK>
__device__ __forceinline__ T wval(const void* w, int64_t gi) {
  if constexpr (WK == 0) return (T)1;
  else if constexpr (WK == 1) return (T) static_cast<const uint32_t*>(w)[gi];
  else return (T) static_cast<const float*>(w)[gi];
}

// ---------------------------------------------------------------- H2
// Donor masks by an 8-neighbour gather, 4 cells per 32-bit SWAR word (no
// atomics; Alg. 1 first loop P:L131-148), and the compacted source queue.
// Ring codes (254/255) never equal a direction, so no bounds tests.
template <class C>
__device__ __forceinline__ void build_masks(Smem<C>& s, int h, int w) {
  const int lane = threadIdx.x & 31;
  const uint32_t* D = reinterpret_cast<const uint32_t*>(s.dirh);
  for (int q = threadIdx.x; q < C::BN / 4; q += C::NT) {
    const int ly = (4 * q) / C::BC, lx = (4 * q) % C::BC;
    const int hw = C::hidx(ly, lx) >> 2;  // word index of the 4 cells
    constexpr int RW = C::HS / 4;
    const uint32_t u0 = D[hw - RW - 1], u1 = D[hw - RW], u2 = D[hw - RW + 1];
    const uint32_t c0 = D[hw - 1], c1 = D[hw], c2 = D[hw + 1];
    const uint32_t d0 = D[hw + RW - 1], d1 = D[hw + RW], d2 = D[hw + RW + 1];
    // neighbour bytes for the 4 cells in each direction (byte j <-> cell j)
    const uint32_t nN = u1, nS = d1;
    const uint32_t nE = __funnelshift_r(c1, c2, 8), nW = __funnelshift_r(c0, c1, 24);
    const uint32_t nNE = __funnelshift_r(u1, u2, 8), nNW = __funnelshift_r(u0, u1, 24);
    const uint32_t nSE = __funnelshift_r(d1, d2, 8), nSW = __funnelshift_r(d0, d1, 24);
    uint32_t m = 0;
    // a neighbour in direction k is a donor iff its code points back: opp(k)
    m |= (__vcmpeq4(nN, 0x05050505u) & 0x01010101u) << 0;   // k=1 N  -> S(5)
    m |= (__vcmpeq4(nNE, 0x06060606u) & 0x01010101u) << 1;  // k=2 NE -> SW(6)
    m |= (__vcmpeq4(nE, 0x07070707u) & 0x01010101u) << 2;   // k=3 E  -> W(7)
    m |= (__vcmpeq4(nSE, 0x08080808u) & 0x01010101u) << 3;  // k=4 SE -> NW(8)
    m |= (__vcmpeq4(nS, 0x01010101u) & 0x01010101u) << 4;   // k=5 S  -> N(1)
    m |= (__vcmpeq4(nSW, 0x02020202u) & 0x01010101u) << 5;  // k=6 SW -> NE(2)
    m |= (__vcmpeq4(nW, 0x03030303u) & 0x01010101u) << 6;   // k=7 W  -> E(3)
    m |= (__vcmpeq4(nNW, 0x04040404u) & 0x01010101u) << 7;  // k=8 NW -> SE(4)
    // NoData (255) and ring cells (254, inside the word when the block is
    // ragged) are not cells of the block: no donors, never sources
    const uint32_t nd = __vcmpgeu4(c1, 0xFEFEFEFEu);
    m &= ~nd;
    s.msk4[q] = m;
    s.pend[q] = m;
    // sources: data cells without in-block donors
    const uint32_t zero = __vcmpeq4(m, 0u) & ~nd;  // 0xFF per source byte
    const uint32_t sb = zero & 0x80808080u;
    const int cnt = __popc(sb);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    uint32_t base = 0;
    if (lane == 31 && total) base = atomicAdd(&s.nsrc, (uint32_t)total);
    base = __shfl_sync(0xFFFFFFFFu, base, 31) + (uint32_t)(incl - cnt);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (sb & (0x80u << (8 * j))) s.src[base++] = (uint16_t)(4 * q + j);
  }
  (void)h;
  (void)w;
}

// ---------------------------------------------------------------- H3
// Walks from the shared source queue (both passes).  On entry dirh, masks,
// pend, src/nsrc and A (= w [+ x]) are set and synced.  Returns the number of
// cells this thread retired.
__device__ __forceinline__ void fence_cta() { asm volatile("fence.acq_rel.cta;" ::: "memory"); }

template <class C, class T>
__device__ __forceinline__ uint32_t chain_follow(Smem<C>& s, T* A) {
  const uint32_t nsrc = s.nsrc;
  uint32_t retired = 0;
  bool live = false;
  int ch = 0, ca = 0, d = 0;
  T a = (T)0;
#ifdef FA_PHASE_CLOCKS
  uint32_t iters = 0;
  struct Tally {
    uint32_t& it;
    const uint32_t& ret;
    __device__ ~Tally() {
      uint32_t mx = it, sm = ret;
      for (int o = 16; o; o >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
        sm += __shfl_xor_sync(0xFFFFFFFFu, sm, o);
      }
      if ((threadIdx.x & 31) == 0) {
        atomicAdd(&g_phase[14], (unsigned long long)mx);
        atomicAdd(&g_phase[15], (unsigned long long)sm);
      }
    }
  } tally{iters, retired};
#endif
  for (;;) {
#ifdef FA_PHASE_CLOCKS
    ++iters;
#endif
    if (!live) {
      // take the next source (per-lane shared atomic; no warp votes, so a
      // lane never waits for the others of its warp)
      const uint32_t q = atomicAdd(&s.qhead, 1u);
      if (q >= nsrc) break;
      ca = s.src[q];
      ch = C::a2h(ca);
      d = s.dirh[ch];
      a = A[ca];
      live = true;
      ++retired;
    }
    // one step downstream
    if (d == kNoFlow || d > 8) { live = false; continue; }
    const int th = ch + C::offH(d);
    const int ta = (ca + C::offA(d)) & (C::BN - 1);  // clamped; unused when the walk stops
    const int dt = s.dirh[th];
    const uint32_t m = s.msk(ta);
    const T at = A[ta];  // w(t) [+ x(t)]: only the walk that finishes t writes A[t]
    if (dt >= kOut) { live = false; continue; }  // leaves the block, or drops into NoData (D8)
    if ((m & (m - 1)) == 0) {
      a = at + a;  // sole in-block donor: no atomic
    } else {
      // junction: clear our bit; the last arrival gathers the donors
      const uint32_t bit = 1u << ((d + 3) & 7);  // bit of the opposite direction
      const int sh = (ta & 3) * 8;
      fence_cta();  // release our value
      const uint32_t old = atomicAnd(&s.pend[ta >> 2], ~(bit << sh));
      if (((old >> sh) & 0xFFu) != bit) { live = false; continue; }  // others pending
      fence_cta();  // acquire the other donors' values
      uint32_t mm = m;
      T acc = at;
      do {  // donors in code order (fixed summation order)
        const int k = __ffs(mm);
        mm &= mm - 1;
        acc = acc + A[ta + C::offA(k)];
      } while (mm);
      a = acc;
    }
    A[ta] = a;
    ch = th;
    ca = ta;
    d = dt;
    ++retired;
  }
  return retired;
}

// ---------------------------------------------------------------- shared stages
template <class C>
__device__ __forceinline__ void init_dirh(Smem<C>& s) {
  uint32_t* D = reinterpret_cast<uint32_t*>(s.dirh);
  for (int i = threadIdx.x; i < C::HN / 4; i += C::NT) D[i] = 0xFFFFFFFFu;
}

// interior directions from global (pass 2 and pass 1 from dirs); bad codes
// -> NoData, flagged when `check`
template <class C>
__device__ __forceinline__ void load_dirs(Smem<C>& s, const uint8_t* dirs, const Geom& g, int64_t y0,
                                          int64_t x0, int h, int w, bool check, uint32_t* status) {
  const bool vec = w == C::BC && ((x0 & 3) == 0) && ((g.W & 3) == 0) &&
                   ((reinterpret_cast<uintptr_t>(dirs) & 3) == 0);
  bool bad = false;
  if (vec) {
    for (int q = threadIdx.x; q < h * (C::BC / 4); q += C::NT) {
      const int ly = q / (C::BC / 4), lx = (q % (C::BC / 4)) * 4;
      uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(dirs + (y0 + ly) * g.W + x0 + lx));
      // bytes > 8 and != 255 are illegal (D1)
      const uint32_t hi = __vcmpgtu4(v, 0x08080808u) & ~__vcmpeq4(v, 0xFFFFFFFFu);
      if (hi) { bad = true; v |= hi; }
      *reinterpret_cast<uint32_t*>(&s.dirh[C::hidx(ly, lx)]) = v;
    }
  } else {
    for (int i = threadIdx.x; i < h * C::BC; i += C::NT) {
      const int ly = i / C::BC, lx = i % C::BC;
      if (lx >= w) continue;
      uint8_t d = dirs[(y0 + ly) * g.W + x0 + lx];
      if (d > 8 && d != kNoData) { bad = true; d = kNoData; }
      s.dirh[C::hidx(ly, lx)] = d;
    }
  }
  if (check && bad) atomicOr(status, ST_BADCODE);
}

// Weights prefetched into registers at kernel entry (full, aligned blocks),
// so their HBM latency overlaps the staging / D8 / mask phases.
template <class C, int WK>
struct WPre {
  static constexpr int R = C::BN / (4 * C::NT);  // 16-byte groups per thread
  uint4 r[WK == 0 ? 1 : R];
  bool vec = false;
  __device__ __forceinline__ void load(const void* wp, const Geom& g, int64_t y0, int64_t x0, int h, int w) {
    if (WK == 0) return;
    vec = h == C::BR && w == C::BC && ((x0 & 3) == 0) && ((g.W & 3) == 0) &&
          ((reinterpret_cast<uintptr_t>(wp) & 15) == 0);
    if (!vec) return;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int q = threadIdx.x + k * C::NT;
      const int ly = q / (C::BC / 4), lx = (q % (C::BC / 4)) * 4;
      r[k] = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint32_t*>(wp) + (y0 + ly) * g.W + x0 + lx));
    }
  }
};

// A = w (Eq. 1; Alg. 1 "A(c) <- A(c) + 1") for data cells
template <class C, class T, int WK>
__device__ __forceinline__ void init_values(Smem<C>& s, T* A, const void* wp, const WPre<C, WK>& pre,
                                            const Geom& g, int64_t y0, int64_t x0, int h, int w,
                                            uint32_t* status, unsigned long long* wsum_out) {
  unsigned long long wsum = 0;
  uint32_t nd = 0;
  bool bad = false;
  // store one group of 4 cells (raw weight bits in u[]) into A
  auto put = [&](int q, const uint32_t u[4], bool have) {
    const int ly = q / (C::BC / 4), lx = (q % (C::BC / 4)) * 4;
    const uint32_t dw = *reinterpret_cast<const uint32_t*>(&s.dirh[C::hidx(ly, lx)]);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool data = ((dw >> (8 * j)) & 0xFF) < kOut;  // excludes NoData and the ring
      if (!data) continue;
      T v;
      if constexpr (WK == 0) {
        v = (T)1;
      } else if constexpr (WK == 1) {
        v = (T)u[j];
      } else {
        const float f = __uint_as_float(u[j]);
        if (!weight_ok<WK>(f)) bad = true;
        v = (T)f;
      }
      (void)have;
      A[ly * C::BC + lx + j] = v;
      ++nd;
      if constexpr (!std::is_same<T, double>::value) wsum += (unsigned long long)v;
    }
  };
  if (WK != 0 && pre.vec) {
#pragma unroll
    for (int k = 0; k < WPre<C, WK>::R; ++k) {
      const uint32_t u[4] = {pre.r[k].x, pre.r[k].y, pre.r[k].z, pre.r[k].w};
      put(threadIdx.x + k * C::NT, u, true);
    }
  } else {
    for (int q = threadIdx.x; q < h * (C::BC / 4); q += C::NT) {
      const int ly = q / (C::BC / 4), lx = (q % (C::BC / 4)) * 4;
      const int64_t gi = (y0 + ly) * g.W + x0 + lx;
      uint32_t u[4] = {0, 0, 0, 0};
      if (WK != 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (lx + j < w) u[j] = static_cast<const uint32_t*>(wp)[gi + j];
      }
      put(q, u, true);
    }
  }
  if (bad) atomicOr(status, ST_BADWEIGHT);
  if (!std::is_same<T, double>::value && wsum_out) {
    for (int o = 16; o; o >>= 1) wsum += __shfl_xor_sync(0xFFFFFFFFu, wsum, o);
    if ((threadIdx.x & 31) == 0 && wsum) atomicAdd(wsum_out, wsum);
  }
  atomicAdd(&s.ndata, nd);
}

// write the block's values A (NoData marker D9), 16-byte stores when aligned
template <class C, class T>
__device__ __forceinline__ void write_block(const Smem<C>& s, const T* A, T* out, const Geom& g, int64_t y0,
                                            int64_t x0, int h, int w) {
  constexpr int V = 16 / sizeof(T);  // cells per 16-byte store
  const bool vec = w == C::BC && ((x0 % V) == 0) && ((g.W % V) == 0) &&
                   ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  if (vec) {
    for (int q = threadIdx.x; q < h * (C::BC / V); q += C::NT) {
      const int ly = q / (C::BC / V), lx = (q % (C::BC / V)) * V;
      alignas(16) T v[V];
#pragma unroll
      for (int j = 0; j < V; ++j)
        v[j] = s.dirh[C::hidx(ly, lx + j)] == kNoData ? AccT<T>::marker() : A[ly * C::BC + lx + j];
      *reinterpret_cast<uint4*>(out + (y0 + ly) * g.W + x0 + lx) = *reinterpret_cast<const uint4*>(v);
    }
  } else {
    for (int i = threadIdx.x; i < h * C::BC; i += C::NT) {
      const int ly = i / C::BC, lx = i % C::BC;
      if (lx >= w) continue;
      const bool nodata = s.dirh[C::hidx(ly, lx)] == kNoData;
      out[(y0 + ly) * g.W + x0 + lx] = nodata ? AccT<T>::marker() : A[i];
    }
  }
}

// ---------------------------------------------------------------- pass 1
template <class C, class T, int WK, bool FROM_DEM>
__global__ void __launch_bounds__(C::NT) k_pass1(PassArgs<T, WK> P) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* A = reinterpret_cast<T*>(smem);
  float* zs = reinterpret_cast<float*>(smem);
  Smem<C>& s = *reinterpret_cast<Smem<C>*>(smem + SmemSize<C, T>::region);
  const Geom& g = P.g;
  const int64_t b = blockIdx.x;
  int64_t y0, x0;
  int h, w;
  g.block_box(b, y0, x0, h, w);
  const int tid = threadIdx.x;
  if (h <= 0 || w <= 0) {
    for (int p = tid; p < C::PB; p += C::NT) P.slot_root[b * C::PB + p] = kNone;
    return;
  }
  PH_T0;
  WPre<C, WK> pre;
  pre.load(P.w, g, y0, x0, h, w);  // in flight during staging, D8 and masks
  if (tid == 0) s.cnt_exit = s.processed = s.ndata = s.nsrc = s.qhead = 0;
  init_dirh(s);
  if (FROM_DEM) {
    // ---- stage z with its halo (NoData and off-grid -> NaN), then D8 (H1)
    // full, aligned blocks: each window row = BC/4 float4 loads + 2 halo
    // scalars; otherwise one scalar per cell (compile-time strides only)
    const bool zvec = w == C::BC && ((x0 & 3) == 0) && ((g.W & 3) == 0) &&
                      ((reinterpret_cast<uintptr_t>(P.dem) & 15) == 0) &&
                      (!P.dem_up || (reinterpret_cast<uintptr_t>(P.dem_up) & 15) == 0) &&
                      (!P.dem_dn || (reinterpret_cast<uintptr_t>(P.dem_dn) & 15) == 0);
    if (zvec) {
      constexpr int Q = C::BC / 4 + 2;  // per window row: BC/4 quads + 2 halo cells
      for (int i = tid; i < (C::BR + 2) * Q; i += C::NT) {
        const int r = i / Q, k = i % Q, ly = r - 1;
        const int64_t gy = y0 + ly;
        const float* row = (ly > h) ? nullptr
                           : gy < 0 ? (gy == -1 ? P.dem_up : nullptr)
                           : gy >= g.H ? (gy == g.H ? P.dem_dn : nullptr)
                                       : P.dem + gy * g.W;
        float* zrow = zs + r * C::ZS;
        if (k < C::BC / 4) {
          float4 v = make_float4(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000),
                                 __int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
          if (row) {
            v = __ldg(reinterpret_cast<const float4*>(row + x0) + k);
            v.x = stage_z(v.x, P.nodata); v.y = stage_z(v.y, P.nodata);
            v.z = stage_z(v.z, P.nodata); v.w = stage_z(v.w, P.nodata);
          }
          zrow[1 + 4 * k] = v.x; zrow[2 + 4 * k] = v.y; zrow[3 + 4 * k] = v.z; zrow[4 + 4 * k] = v.w;
        } else {
          const int lx = k == C::BC / 4 ? -1 : C::BC;
          const int64_t gx = x0 + lx;
          float v = __int_as_float(0x7fc00000);
          if (row && gx >= 0 && gx < g.W) v = stage_z(row[gx], P.nodata);
          zrow[lx + 1] = v;
        }
      }
    } else {
      for (int i = tid; i < C::ZN; i += C::NT) {
        const int ly = i / C::ZS - 1, lx = i % C::ZS - 1;
        float v = __int_as_float(0x7fc00000);
        if (ly <= h && lx <= w) {
          const int64_t gy = y0 + ly, gx = x0 + lx;
          if (gx >= 0 && gx < g.W) {
            const float* row = gy < 0 ? P.dem_up : gy >= g.H ? P.dem_dn : P.dem + gy * g.W;
            if (row && gy >= -1 && gy <= g.H) v = stage_z(row[gx], P.nodata);
          }
        }
        zs[i] = v;
      }
    }
    __syncthreads();
    PH_MARK(8);
    // D8 for the block's cells, 4 per thread: one 32-bit shared store and one
    // 32-bit global store of the packed codes
    for (int q = tid; q < C::BN / 4; q += C::NT) {
      const int ly = (4 * q) / C::BC, lx = (4 * q) % C::BC;
      if (ly >= h) continue;
      uint32_t packed = 0xFFFFFFFFu;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (lx + j < w) {
          const uint32_t code = d8_code<C::ZS>(zs, (ly + 1) * C::ZS + lx + j + 1);
          packed = (packed & ~(0xFFu << (8 * j))) | (code << (8 * j));
        }
      *reinterpret_cast<uint32_t*>(&s.dirh[C::hidx(ly, lx)]) = packed;
      if (P.dirs_out) {
        uint8_t* dst = P.dirs_out + (y0 + ly) * g.W + x0 + lx;
        if (lx + 3 < w && (reinterpret_cast<uintptr_t>(dst) & 3) == 0) {
          *reinterpret_cast<uint32_t*>(dst) = packed;
        } else {
          for (int j = 0; j < 4 && lx + j < w; ++j) dst[j] = (uint8_t)(packed >> (8 * j));
        }
      }
    }
    __syncthreads();
    // halo ring: NoData-ness only (after the packed stores, which may cover it)
    const int rn = 2 * (w + 2) + 2 * h;
    for (int i = tid; i < rn; i += C::NT) {
      int ly, lx;
      if (i < w + 2) { ly = -1; lx = i - 1; }
      else if (i < 2 * (w + 2)) { ly = h; lx = i - (w + 2) - 1; }
      else { const int j = i - 2 * (w + 2); ly = j >> 1; lx = (j & 1) ? w : -1; }
      s.dirh[C::hidx(ly, lx)] = isnan(zs[(ly + 1) * C::ZS + lx + 1]) ? kNoData : kOut;
    }
    __syncthreads();  // zs dead from here on; A aliases it
    PH_MARK(9);
  } else {
    __syncthreads();
    load_dirs<C>(s, P.dirs_in, g, y0, x0, h, w, true, P.status);
    // halo ring: 254 for data outside the block, 255 for NoData / off-grid
    const int rn = 2 * (w + 2) + 2 * h;
    for (int i = tid; i < rn; i += C::NT) {
      int ly, lx;
      if (i < w + 2) { ly = -1; lx = i - 1; }
      else if (i < 2 * (w + 2)) { ly = h; lx = i - (w + 2) - 1; }
      else { const int j = i - 2 * (w + 2); ly = j >> 1; lx = (j & 1) ? w : -1; }
      const int64_t gy = y0 + ly, gx = x0 + lx;
      uint8_t code = kNoData;
      if (gx >= 0 && gx < g.W) {
        const uint8_t* row = gy < 0 ? P.dirs_up : gy >= g.H ? P.dirs_dn : P.dirs_in + gy * g.W;
        if (row && gy >= -1 && gy <= g.H && row[gx] != kNoData) code = kOut;
      }
      s.dirh[C::hidx(ly, lx)] = code;
    }
    __syncthreads();
  }
  build_masks<C>(s, h, w);
  init_values<C, T, WK>(s, A, P.w, pre, g, y0, x0, h, w, P.status, P.wsum);
  __syncthreads();
  PH_MARK(10);
  const uint32_t ret = chain_follow<C, T>(s, A);
  atomicAdd(&s.processed, ret);
  __syncthreads();
  PH_MARK(11);
  if (tid == 0 && s.processed != s.ndata) atomicOr(P.status, ST_CYCLE);
  // RETAIN: the block-local accumulation goes straight to the output;
  // pass 2 then only adds the offsets along the entry paths (k_retain)
  if (P.retain) write_block<C, T>(s, A, P.acc, g, y0, x0, h, w);
  // ---- H4: block exits -> graph nodes (compacted), perimeter links
  const int np = (int)perim_count(h, w);
  for (int p = tid; p < C::PB; p += C::NT) {
    uint32_t r = kNone;
    if (p < np) {
      int64_t px, py;
      perim_xy(p, h, w, px, py);
      const int d = s.dirh[C::hidx((int)py, (int)px)];
      if (d >= 1 && d <= 8) {
        const int ty = (int)py + dir_dy(d), tx = (int)px + dir_dx(d);
        if ((unsigned)ty >= (unsigned)h || (unsigned)tx >= (unsigned)w) r = atomicAdd(&s.cnt_exit, 1u);
      }
    }
    s.slot_nid[p] = r;  // rank among the block's exits, for now
  }
  __syncthreads();
  if (tid == 0) s.base = s.cnt_exit ? atomicAdd(P.node_count, s.cnt_exit) : 0;
  __syncthreads();
  int64_t t0y, t0x, th, tw;
  g.tile_box(g.tile_of_block(b), t0y, t0x, th, tw);
  for (int p = tid; p < np; p += C::NT) {
    const uint32_t rank = s.slot_nid[p];
    if (rank == kNone) continue;
    const uint32_t nid = s.base + rank;
    int64_t px, py;
    perim_xy(p, h, w, px, py);
    const int d = s.dirh[C::hidx((int)py, (int)px)];
    const int ty = (int)py + dir_dy(d), tx = (int)px + dir_dx(d);
    const bool dead = s.dirh[C::hidx(ty, tx)] == kNoData;
    const int64_t gy = y0 + ty, gx = x0 + tx;
    uint8_t fl = dead ? NF_DEAD : 0;
    if (gy < t0y || gx < t0x || gy >= t0y + th || gx >= t0x + tw) fl |= NF_OUT_TILE;
    uint32_t tgt = kNone;  // none: dropped, or in another strip (carried by the tile records)
    if (!dead && gy >= 0 && gy < g.H) {
      int tly, tlx;
      const int64_t tb = g.block_of(gy, gx, tly, tlx);
      int64_t by0, bx0;
      int bh, bw;
      g.block_box(tb, by0, bx0, bh, bw);
      tgt = (uint32_t)(tb * C::PB + perim_index(tlx, tly, bh, bw));
    }
    P.node_val[nid] = A[py * C::BC + px];
    P.node_slot[nid] = (uint32_t)(b * C::PB + p);
    P.node_tgt[nid] = tgt;
    P.node_flags[nid] = fl;
    s.slot_nid[p] = nid;
  }
  __syncthreads();
  PH_MARK(12);
  // Alg. 2 FollowPath for every block perimeter cell (root exit node or none)
  for (int p = tid; p < C::PB; p += C::NT) {
    uint32_t root = kNone;
    if (p < np) {
      int64_t cx, cy;
      perim_xy(p, h, w, cx, cy);
      int ly = (int)cy, lx = (int)cx;
      for (int steps = 0; steps <= h * w; ++steps) {
        const int dd = s.dirh[C::hidx(ly, lx)];
        if (dd == kNoFlow || dd > 8) break;  // FlowTerminates (NoFlow)
        const int ny = ly + dir_dy(dd), nx = lx + dir_dx(dd);
        if ((unsigned)ny >= (unsigned)h || (unsigned)nx >= (unsigned)w) {
          root = s.slot_nid[perim_index(lx, ly, h, w)];  // (ly, lx) is a block exit
          break;
        }
        if (s.dirh[C::hidx(ny, nx)] == kNoData) break;  // terminates in in-block NoData
        ly = ny;
        lx = nx;
      }
    }
    P.slot_root[b * C::PB + p] = root;
  }
  __syncthreads();
  PH_MARK(13);
}

// ---------------------------------------------------------------- pass 2
template <class C, class T, int WK>
__global__ void __launch_bounds__(C::NT) k_pass2(PassArgs<T, WK> P) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* A = reinterpret_cast<T*>(smem);
  Smem<C>& s = *reinterpret_cast<Smem<C>*>(smem + SmemSize<C, T>::region);
  const Geom& g = P.g;
  const int64_t b = blockIdx.x;
  int64_t y0, x0;
  int h, w;
  g.block_box(b, y0, x0, h, w);
  if (h <= 0 || w <= 0) return;
  const int tid = threadIdx.x;
  PH_T0;
  WPre<C, WK> pre;
  pre.load(P.w, g, y0, x0, h, w);  // in flight during staging and masks
  if (tid == 0) s.processed = s.ndata = s.nsrc = s.qhead = 0;
  init_dirh(s);  // ring = 255: never a donor, stops walks
  __syncthreads();
  load_dirs<C>(s, P.dirs_in, g, y0, x0, h, w, false, P.status);
  __syncthreads();
  PH_MARK(0);
  build_masks<C>(s, h, w);
  __syncthreads();
  PH_MARK(1);
  init_values<C, T, WK>(s, A, P.w, pre, g, y0, x0, h, w, P.status, nullptr);
  __syncthreads();
  PH_MARK(2);
  // inject x at the block perimeter (offset propagation; D12)
  const int np = (int)perim_count(h, w);
  for (int p = tid; p < np; p += C::NT) {
    int64_t px, py;
    perim_xy(p, h, w, px, py);
    if (s.dirh[C::hidx((int)py, (int)px)] == kNoData) continue;
    const T x = P.x_slot[b * C::PB + p];
    A[py * C::BC + px] = A[py * C::BC + px] + x;
  }
  __syncthreads();
  PH_MARK(3);
  const uint32_t ret = chain_follow<C, T>(s, A);
  atomicAdd(&s.processed, ret);
  __syncthreads();
  PH_MARK(4);
  if (tid == 0 && s.processed != s.ndata) atomicOr(P.status, ST_CYCLE);
  write_block<C, T>(s, A, P.acc, g, y0, x0, h, w);
  PH_MARK(5);
}

// ---------------------------------------------------------------- RETAIN finalize
// "add A' to every cell in its downstream flow path" (Alg. 3): one
// thread per block entry slot with a non-zero offset x walks the entry's
// in-block path, adding x to every cell up to the block exit (or the NoFlow
// terminal; flow into NoData is dropped).  acc already holds the block-local
// accumulation written by pass 1, so A = A_blk + sum of the offsets whose path
// passes the cell (linearity, D12).  Offsets on shared path segments sum.
template <class T>
__global__ void __launch_bounds__(256) k_retain(Geom g, const T* __restrict__ x_slot,
                                                const uint8_t* __restrict__ dirs, T* acc) {
  const int64_t nslots = g.nblocks * g.pb;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslots;
       s += (int64_t)gridDim.x * blockDim.x) {
    const T x = x_slot[s];
    if (x == (T)0) continue;
    const uint32_t b = (uint32_t)s / (uint32_t)g.pb, p = (uint32_t)s - b * (uint32_t)g.pb;
    int64_t y0, x0;
    int h, w;
    g.block_box(b, y0, x0, h, w);
    if (p >= (uint32_t)perim_count(h, w)) continue;
    int64_t px, py;
    perim_xy(p, h, w, px, py);
    int ly = (int)py, lx = (int)px;
    int64_t gi = (y0 + ly) * g.W + x0 + lx;
    int d = __ldg(dirs + gi);
    for (int steps = 0; steps <= h * w; ++steps) {
      atomic_add(&acc[gi], x);
      if (d == kNoFlow || d > 8) break;
      const int ny = ly + dir_dy(d), nx = lx + dir_dx(d);
      if ((unsigned)ny >= (unsigned)h || (unsigned)nx >= (unsigned)w) break;  // leaves the block
      const int64_t ni = gi + dir_dy(d) * g.W + dir_dx(d);
      const int nd = __ldg(dirs + ni);
      if (nd == kNoData) break;  // dropped (D8)
      ly = ny;
      lx = nx;
      gi = ni;
      d = nd;
    }
  }
}

template <class T>
cudaError_t launch_retain(const Geom& g, const T* x_slot, const uint8_t* dirs, T* acc, cudaStream_t st) {
  const int64_t n = g.nblocks * g.pb;
  int64_t grid = (n + 255) / 256;
  if (grid > 148 * 32) grid = 148 * 32;
  k_retain<T><<<(unsigned)(grid < 1 ? 1 : grid), 256, 0, st>>>(g, x_slot, dirs, acc);
  return cudaGetLastError();
}
template cudaError_t launch_retain<uint32_t>(const Geom&, const uint32_t*, const uint8_t*, uint32_t*, cudaStream_t);
template cudaError_t launch_retain<unsigned long long>(const Geom&, const unsigned long long*, const uint8_t*,
                                                       unsigned long long*, cudaStream_t);
template cudaError_t launch_retain<double>(const Geom&, const double*, const uint8_t*, double*, cudaStream_t);

// ---------------------------------------------------------------- launchers
template <class C, class T, int WK>
cudaError_t launch_pass1_c(const PassArgs<T, WK>& a, bool from_dem, cudaStream_t st) {
  const size_t sm = SmemSize<C, T>::total;
  if (from_dem) {
    auto k = k_pass1<C, T, WK, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<(unsigned)a.g.nblocks, C::NT, sm, st>>>(a);
  } else {
    auto k = k_pass1<C, T, WK, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<(unsigned)a.g.nblocks, C::NT, sm, st>>>(a);
  }
  return cudaGetLastError();
}

template <class C, class T, int WK>
cudaError_t launch_pass2_c(const PassArgs<T, WK>& a, cudaStream_t st) {
  const size_t sm = SmemSize<C, T>::total;
  auto k = k_pass2<C, T, WK>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k<<<(unsigned)a.g.nblocks, C::NT, sm, st>>>(a);
  return cudaGetLastError();
}

using Cfg32 = Cfg<32, 32, 2>;
using Cfg32w1 = Cfg<32, 32, 1>;
using Cfg32w4 = Cfg<32, 32, 4>;
using Cfg3264 = Cfg<32, 64, 2>;
using Cfg64 = Cfg<64, 64, 4>;
using Cfg64w1 = Cfg<64, 64, 1>;
using Cfg64w2 = Cfg<64, 64, 2>;

template <class T, int WK>
cudaError_t launch_pass1(const PassArgs<T, WK>& a, bool from_dem, cudaStream_t st) {
  if (a.g.br == 32 && a.g.bc == 32 && a.g.nw == 1) return launch_pass1_c<Cfg32w1, T, WK>(a, from_dem, st);
  if (a.g.br == 32 && a.g.bc == 32 && a.g.nw == 4) return launch_pass1_c<Cfg32w4, T, WK>(a, from_dem, st);
  if (a.g.br == 32 && a.g.bc == 32) return launch_pass1_c<Cfg32, T, WK>(a, from_dem, st);
  if (a.g.br == 32 && a.g.bc == 64) return launch_pass1_c<Cfg3264, T, WK>(a, from_dem, st);
  if (a.g.br == 64 && a.g.bc == 64 && a.g.nw == 1) return launch_pass1_c<Cfg64w1, T, WK>(a, from_dem, st);
  if (a.g.br == 64 && a.g.bc == 64 && a.g.nw == 2) return launch_pass1_c<Cfg64w2, T, WK>(a, from_dem, st);
  if (a.g.br == 64 && a.g.bc == 64) return launch_pass1_c<Cfg64, T, WK>(a, from_dem, st);
  return cudaErrorInvalidValue;
}

template <class T, int WK>
cudaError_t launch_pass2(const PassArgs<T, WK>& a, cudaStream_t st) {
  if (a.g.br == 32 && a.g.bc == 32 && a.g.nw == 1) return launch_pass2_c<Cfg32w1, T, WK>(a, st);
  if (a.g.br == 32 && a.g.bc == 32 && a.g.nw == 4) return launch_pass2_c<Cfg32w4, T, WK>(a, st);
  if (a.g.br == 32 && a.g.bc == 32) return launch_pass2_c<Cfg32, T, WK>(a, st);
  if (a.g.br == 32 && a.g.bc == 64) return launch_pass2_c<Cfg3264, T, WK>(a, st);
  if (a.g.br == 64 && a.g.bc == 64 && a.g.nw == 1) return launch_pass2_c<Cfg64w1, T, WK>(a, st);
  if (a.g.br == 64 && a.g.bc == 64 && a.g.nw == 2) return launch_pass2_c<Cfg64w2, T, WK>(a, st);
  if (a.g.br == 64 && a.g.bc == 64) return launch_pass2_c<Cfg64, T, WK>(a, st);
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

// ---------------------------------------------------------------- standalone D8 (fa_flowdirs)
constexpr int DR = 32, DC = 128;  // output tile per CTA
__global__ void __launch_bounds__(256) k_d8(const float* __restrict__ dem, int64_t H, int64_t W,
                                            float nodata, uint8_t* __restrict__ dirs) {
  __shared__ float zs[(DR + 2) * (DC + 2)];
  const int64_t y0 = (int64_t)blockIdx.y * DR, x0 = (int64_t)blockIdx.x * DC;
  for (int i = threadIdx.x; i < (DR + 2) * (DC + 2); i += 256) {
    const int ly = i / (DC + 2) - 1, lx = i % (DC + 2) - 1;
    const int64_t gy = y0 + ly, gx = x0 + lx;
    float v = __int_as_float(0x7fc00000);
    if (gy >= 0 && gx >= 0 && gy < H && gx < W) v = stage_z(dem[gy * W + gx], nodata);
    zs[i] = v;
  }
  __syncthreads();
  // each thread: 4 consecutive cells of one row -> one 32-bit store when aligned
  for (int q = threadIdx.x; q < DR * DC / 4; q += 256) {
    const int ly = q / (DC / 4), lx = (q % (DC / 4)) * 4;
    const int64_t gy = y0 + ly, gx = x0 + lx;
    if (gy >= H) continue;
    uint32_t packed = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint8_t c = d8_code<DC + 2>(zs, (ly + 1) * (DC + 2) + lx + j + 1);
      packed |= (uint32_t)c << (8 * j);
    }
    const int64_t gi = gy * W + gx;
    if (gx + 3 < W && (gi & 3) == 0) {
      *reinterpret_cast<uint32_t*>(dirs + gi) = packed;
    } else {
      for (int j = 0; j < 4; ++j)
        if (gx + j < W) dirs[gi + j] = (uint8_t)(packed >> (8 * j));
    }
  }
}

cudaError_t launch_d8(const float* dem, int64_t H, int64_t W, float nodata, uint8_t* dirs,
                      cudaStream_t st) {
  dim3 grid((unsigned)((W + DC - 1) / DC), (unsigned)((H + DR - 1) / DR));
  k_d8<<<grid, 256, 0, st>>>(dem, H, W, nodata, dirs);
  return cudaGetLastError();
}

}  // namespace fa
