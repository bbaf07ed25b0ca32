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
// H3 scheduling (differs from the paper's FIFO): chain
// following.  Every source (no in-block donor) starts a walk; a walk adds its
// value into the next cell and continues while it is that cell's only pending
// donor.  Cells with exactly one donor need no atomic at all; at a junction the
// arriving walk clears its bit in the target's pending-donor mask with one
// shared-memory atomicAnd, and the last arrival gathers the donors' finished
// values (fixed donor order) and continues.  Work is O(1) per cell; the
// critical path is the longest in-block flow path.
#include "fa_internal.cuh"

namespace fa {

constexpr int HS = BC + 2;             // halo'd row stride
constexpr int HN = (BR + 2) * (BC + 2);  // halo'd cells


struct __align__(16) SmemCommon {
  uint8_t dirh[HN];   // directions with a 1-cell halo ring (ring: 255 = NoData/off-grid)
  uint8_t msk[BN];    // in-block donor mask: bit k-1 set if neighbour in direction k drains here
  uint32_t pend[BN / 4];  // pending-donor masks, 4 cells per word (atomicAnd)
  uint32_t slot_nid[PB];
  uint32_t cnt_exit, base, processed, ndata;
};

template <class T>
struct SmemSize {
  static constexpr size_t a_bytes = sizeof(T) * BN;
  static constexpr size_t z_bytes = sizeof(float) * HN;
  static constexpr size_t region = ((a_bytes > z_bytes ? a_bytes : z_bytes) + 15) / 16 * 16;
  static constexpr size_t total = region + sizeof(SmemCommon);
};

template <int WK>
__device__ __forceinline__ bool load_weight(const void* w, int64_t gi, double& wd, unsigned long long& wu) {
  if (WK == 0) {
    wd = 1.0;
    wu = 1;
    return true;
  } else if (WK == 1) {
    uint32_t v = static_cast<const uint32_t*>(w)[gi];
    wd = (double)v;
    wu = v;
    return true;
  } else {
    float v = static_cast<const float*>(w)[gi];
    wd = (double)v;
    wu = 0;
    return isfinite(v) && v >= 0.0f;  // D21
  }
}

template <class T>
__device__ __forceinline__ T from_w(double wd, unsigned long long wu) {
  if constexpr (std::is_same<T, double>::value) return wd;
  else return (T)wu;
}

// In-block accumulation by chain following (shared by both passes).  On
// entry: dirh, msk, pend and A (= w [+ x]) are set and synced.  Returns the
// number of cells this thread retired.
//
// One flat loop per lane: when a lane's walk ends it immediately starts its
// next source, so lanes of a warp never wait for each other between walks
// (a per-source loop would make every warp pay the sum over its sources of
// the longest walk among its 32 lanes).  Each step issues its three shared
// loads (direction, donor mask, value of the next cell) together.
template <class T>
__device__ __forceinline__ uint32_t chain_follow(SmemCommon& s, T* A, int h, int w) {
  uint32_t retired = 0;
  int next = threadIdx.x;  // next candidate source of this lane
  int ly = 0, lx = 0, d = kNoFlow;
  bool live = false;
  T a = (T)0;
  for (;;) {
    if (!live) {
      // fetch this lane's next source (data cell without in-block donors)
      while (next < BN) {
        const int i = next;
        next += kThreads;
        const int y = i / BC, x = i % BC;
        if (y >= h || x >= w) continue;
        const int dd = s.dirh[(y + 1) * HS + x + 1];
        if (dd == kNoData || s.msk[i] != 0) continue;
        ly = y;
        lx = x;
        d = dd;
        a = A[i];
        live = true;
        ++retired;
        break;
      }
      if (!live) break;
    }
    // one step of the walk from (ly, lx) with direction d and value a
    if (d == kNoFlow || d > 8) { live = false; continue; }
    const int ty = ly + dir_dy(d), tx = lx + dir_dx(d);
    if ((unsigned)ty >= (unsigned)h || (unsigned)tx >= (unsigned)w) { live = false; continue; }
    const int t = ty * BC + tx;
    const int dt = s.dirh[(ty + 1) * HS + tx + 1];
    const uint32_t m = s.msk[t];
    const T at = A[t];  // w(t) [+ x(t)]: only the walk that finishes t writes A[t]
    if (dt == kNoData) { live = false; continue; }  // dropped into NoData (D8)
    if ((m & (m - 1)) == 0) {
      a = at + a;  // sole in-block donor: no atomic needed
    } else {
      const uint32_t bit = 1u << (dir_opp(d) - 1);
      const int sh = (t & 3) * 8;
      __threadfence_block();  // release our A[c]
      const uint32_t old = atomicAnd(&s.pend[t >> 2], ~(bit << sh));
      if (((old >> sh) & 0xFFu) != bit) { live = false; continue; }  // others pending
      __threadfence_block();  // acquire the other donors' values
      T acc = at;
#pragma unroll
      for (int k = 1; k <= 8; ++k)
        if (m & (1u << (k - 1))) acc = acc + A[(ty + dir_dy(k)) * BC + tx + dir_dx(k)];
      a = acc;
    }
    A[t] = a;
    ly = ty;
    lx = tx;
    d = dt;
    ++retired;
  }
  return retired;
}

// donor masks by gather (H2, Alg. 1 first loop P:L131-148, no atomics)
__device__ __forceinline__ void build_masks(SmemCommon& s, int h, int w) {
  for (int i = threadIdx.x; i < BN; i += kThreads) {
    const int ly = i / BC, lx = i % BC;
    uint32_t m = 0;
    if (ly < h && lx < w && s.dirh[(ly + 1) * HS + lx + 1] != kNoData) {
#pragma unroll
      for (int k = 1; k <= 8; ++k) {
        const int ny = ly + dir_dy(k), nx = lx + dir_dx(k);
        if ((unsigned)ny < (unsigned)h && (unsigned)nx < (unsigned)w &&
            s.dirh[(ny + 1) * HS + nx + 1] == dir_opp(k))
          m |= 1u << (k - 1);
      }
    }
    s.msk[i] = (uint8_t)m;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < BN / 4; i += kThreads) {
    const uint32_t* m4 = reinterpret_cast<const uint32_t*>(s.msk);
    s.pend[i] = m4[i];
  }
}

template <class T, int WK, bool FROM_DEM>
__global__ void __launch_bounds__(kThreads) k_pass1(PassArgs<T, WK> P) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* A = reinterpret_cast<T*>(smem);
  float* zs = reinterpret_cast<float*>(smem);
  SmemCommon& s = *reinterpret_cast<SmemCommon*>(smem + SmemSize<T>::region);
  const Geom& g = P.g;
  const int64_t b = blockIdx.x;
  int64_t y0, x0;
  int h, w;
  g.block_box(b, y0, x0, h, w);
  const int tid = threadIdx.x;
  if (h <= 0 || w <= 0) {
    for (int p = tid; p < PB; p += kThreads) P.slot_root[b * PB + p] = kNone;
    return;
  }
  if (tid == 0) { s.cnt_exit = 0; s.processed = 0; s.ndata = 0; }
  // ---- stage the block + halo ring
  for (int i = tid; i < HN; i += kThreads) {
    s.dirh[i] = kNoData;
    if (FROM_DEM) zs[i] = __int_as_float(0x7fc00000);
  }
  __syncthreads();
  const int rw = w + 2, rn = (h + 2) * (w + 2);
  for (int i = tid; i < rn; i += kThreads) {
    const int ly = i / rw - 1, lx = i % rw - 1;
    const int64_t gy = y0 + ly, gx = x0 + lx;
    const bool in = gy >= 0 && gx >= 0 && gy < g.H && gx < g.W;
    const int hi = (ly + 1) * HS + lx + 1;
    if (FROM_DEM) {
      if (in) zs[hi] = stage_z(P.dem[gy * g.W + gx], P.nodata);
    } else if (in) {
      uint8_t d = P.dirs_in[gy * g.W + gx];
      const bool inner = ly >= 0 && lx >= 0 && ly < h && lx < w;
      if (d > 8 && d != kNoData) {
        if (inner) atomicOr(P.status, ST_BADCODE);
        d = kNoData;
      }
      s.dirh[hi] = d;
    }
  }
  __syncthreads();
  if (FROM_DEM) {
    // H1: D8 for the block's cells; the halo ring only records NoData-ness
    for (int i = tid; i < rn; i += kThreads) {
      const int ly = i / rw - 1, lx = i % rw - 1;
      const int hi = (ly + 1) * HS + lx + 1;
      const bool inner = ly >= 0 && lx >= 0 && ly < h && lx < w;
      if (inner) {
        const uint8_t code = d8_code<HS>(zs, hi);
        s.dirh[hi] = code;
        if (P.dirs_out) P.dirs_out[(y0 + ly) * g.W + x0 + lx] = code;
      } else {
        s.dirh[hi] = isnan(zs[hi]) ? kNoData : (uint8_t)kNoFlow;
      }
    }
    __syncthreads();  // zs dead from here on; A aliases it
  }
  build_masks(s, h, w);
  // ---- A = w (Eq. 1; Alg. 1 "A(c) <- A(c) + 1")
  unsigned long long wsum = 0;
  uint32_t nd = 0;
  for (int i = tid; i < BN; i += kThreads) {
    const int ly = i / BC, lx = i % BC;
    if (ly >= h || lx >= w) continue;
    if (s.dirh[(ly + 1) * HS + lx + 1] == kNoData) continue;
    double wd;
    unsigned long long wu;
    if (!load_weight<WK>(P.w, (y0 + ly) * g.W + x0 + lx, wd, wu)) atomicOr(P.status, ST_BADWEIGHT);
    A[i] = from_w<T>(wd, wu);
    wsum += wu;
    ++nd;
  }
  if (!std::is_same<T, double>::value && P.wsum) {
    for (int o = 16; o; o >>= 1) wsum += __shfl_xor_sync(0xFFFFFFFFu, wsum, o);
    if ((tid & 31) == 0 && wsum) atomicAdd(P.wsum, wsum);
  }
  atomicAdd(&s.ndata, nd);
  __syncthreads();
  // ---- H3
  const uint32_t ret = chain_follow<T>(s, A, h, w);
  atomicAdd(&s.processed, ret);
  __syncthreads();
  if (tid == 0 && s.processed != s.ndata) atomicOr(P.status, ST_CYCLE);
  // ---- H4: block exits -> graph nodes (compacted), perimeter links
  const int np = (int)perim_count(h, w);
  int64_t px = 0, py = 0;
  bool is_exit = false;
  int rank = 0, d = 0;
  if (tid < np) {
    perim_xy(tid, h, w, px, py);
    d = s.dirh[(py + 1) * HS + px + 1];
    if (d >= 1 && d <= 8) {
      const int ty = (int)py + dir_dy(d), tx = (int)px + dir_dx(d);
      is_exit = (unsigned)ty >= (unsigned)h || (unsigned)tx >= (unsigned)w;
    }
    if (is_exit) rank = atomicAdd(&s.cnt_exit, 1u);
  }
  __syncthreads();
  if (tid == 0) s.base = s.cnt_exit ? atomicAdd(P.node_count, s.cnt_exit) : 0;
  __syncthreads();
  if (tid < np) {
    uint32_t nid = kNone;
    if (is_exit) {
      nid = s.base + rank;
      const int ty = (int)py + dir_dy(d), tx = (int)px + dir_dx(d);
      const bool dead = s.dirh[(ty + 1) * HS + tx + 1] == kNoData;
      const int64_t gy = y0 + ty, gx = x0 + tx;
      uint8_t fl = dead ? NF_DEAD : 0;
      int64_t t0y, t0x, th, tw;
      g.tile_box(g.tile_of_block(b), t0y, t0x, th, tw);
      if (gy < t0y || gx < t0x || gy >= t0y + th || gx >= t0x + tw) fl |= NF_OUT_TILE;
      uint32_t tgt = kNone;
      if (!dead) {
        int tly, tlx;
        const int64_t tb = g.block_of(gy, gx, tly, tlx);
        int64_t by0, bx0;
        int bh, bw;
        g.block_box(tb, by0, bx0, bh, bw);
        tgt = (uint32_t)(tb * PB + perim_index(tlx, tly, bh, bw));
      }
      P.node_val[nid] = A[py * BC + px];
      P.node_slot[nid] = (uint32_t)(b * PB + tid);
      P.node_tgt[nid] = tgt;
      P.node_flags[nid] = fl;
    }
    s.slot_nid[tid] = nid;
  }
  __syncthreads();
  for (int p = tid; p < PB; p += kThreads) {
    uint32_t root = kNone;
    if (p < np) {
      int64_t cx, cy;
      perim_xy(p, h, w, cx, cy);
      for (int steps = 0; steps <= h * w; ++steps) {
        const int dd = s.dirh[(cy + 1) * HS + cx + 1];
        if (dd == kNoFlow || dd > 8) break;  // FlowTerminates
        const int ny = (int)cy + dir_dy(dd), nx = (int)cx + dir_dx(dd);
        if ((unsigned)ny >= (unsigned)h || (unsigned)nx >= (unsigned)w) {
          root = s.slot_nid[perim_index(cx, cy, h, w)];
          break;
        }
        if (s.dirh[(ny + 1) * HS + nx + 1] == kNoData) break;  // terminates in NoData
        cx = nx;
        cy = ny;
      }
    }
    P.slot_root[b * PB + p] = root;
  }
}

template <class T, int WK>
__global__ void __launch_bounds__(kThreads) k_pass2(PassArgs<T, WK> P) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* A = reinterpret_cast<T*>(smem);
  SmemCommon& s = *reinterpret_cast<SmemCommon*>(smem + SmemSize<T>::region);
  const Geom& g = P.g;
  const int64_t b = blockIdx.x;
  int64_t y0, x0;
  int h, w;
  g.block_box(b, y0, x0, h, w);
  if (h <= 0 || w <= 0) return;
  const int tid = threadIdx.x;
  if (tid == 0) { s.processed = 0; s.ndata = 0; }
  for (int i = tid; i < HN; i += kThreads) s.dirh[i] = kNoData;
  __syncthreads();
  for (int i = tid; i < BN; i += kThreads) {
    const int ly = i / BC, lx = i % BC;
    if (ly >= h || lx >= w) continue;
    uint8_t d = P.dirs_in[(y0 + ly) * g.W + x0 + lx];
    if (d > 8) d = kNoData;  // codes were validated in pass 1
    s.dirh[(ly + 1) * HS + lx + 1] = d;
  }
  __syncthreads();
  build_masks(s, h, w);
  uint32_t nd = 0;
  for (int i = tid; i < BN; i += kThreads) {
    const int ly = i / BC, lx = i % BC;
    if (ly >= h || lx >= w) continue;
    if (s.dirh[(ly + 1) * HS + lx + 1] == kNoData) continue;
    double wd;
    unsigned long long wu;
    load_weight<WK>(P.w, (y0 + ly) * g.W + x0 + lx, wd, wu);
    A[i] = from_w<T>(wd, wu);
    ++nd;
  }
  atomicAdd(&s.ndata, nd);
  __syncthreads();
  // inject x at the block perimeter (offset propagation; D12)
  const int np = (int)perim_count(h, w);
  for (int p = tid; p < np; p += kThreads) {
    int64_t px, py;
    perim_xy(p, h, w, px, py);
    if (s.dirh[(py + 1) * HS + px + 1] == kNoData) continue;
    const T x = P.x_slot[b * PB + p];
    A[py * BC + px] = A[py * BC + px] + x;
  }
  __syncthreads();
  const uint32_t ret = chain_follow<T>(s, A, h, w);
  atomicAdd(&s.processed, ret);
  __syncthreads();
  if (tid == 0 && s.processed != s.ndata) atomicOr(P.status, ST_CYCLE);
  for (int i = tid; i < BN; i += kThreads) {
    const int ly = i / BC, lx = i % BC;
    if (ly >= h || lx >= w) continue;
    const bool nodata = s.dirh[(ly + 1) * HS + lx + 1] == kNoData;
    P.acc[(y0 + ly) * g.W + x0 + lx] = nodata ? AccT<T>::marker() : A[i];
  }
}

// ---------------------------------------------------------------- launchers
template <class T, int WK>
cudaError_t launch_pass1(const PassArgs<T, WK>& a, bool from_dem, cudaStream_t st) {
  const size_t sm = SmemSize<T>::total;
  if (from_dem) {
    auto k = k_pass1<T, WK, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<(unsigned)a.g.nblocks, kThreads, sm, st>>>(a);
  } else {
    auto k = k_pass1<T, WK, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<(unsigned)a.g.nblocks, kThreads, sm, st>>>(a);
  }
  return cudaGetLastError();
}

template <class T, int WK>
cudaError_t launch_pass2(const PassArgs<T, WK>& a, cudaStream_t st) {
  const size_t sm = SmemSize<T>::total;
  auto k = k_pass2<T, WK>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k<<<(unsigned)a.g.nblocks, kThreads, sm, st>>>(a);
  return cudaGetLastError();
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
