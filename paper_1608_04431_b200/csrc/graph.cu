// graph.cu -- block-exit graph G1, the tile perimeter records and the paper's
// global perimeter graph G2.
//
// Nodes of G1 are the block exit cells written by pass 1 (one per block
// perimeter cell whose direction leaves its block, Alg. 2 "FlowExternal" at
// block level).  parent(e) = the exit reached in the target's block by the
// target cell's in-block path (slot_root), i.e. the paper's producer graph
// ("adjoining edges (or corners)") with the entry->exit links of
// Alg. 2 composed in.  Cutting the edges that leave a paper tile gives the
// per-tile problem (Alg. 1 on the tile): its solution A_T and the
// tile roots give the tile perimeter records (F, A, L per perimeter cell,
// P:L213).  G2 is then built from those records exactly as the paper's
// producer does and solved with the same forest primitive; the
// returned offsets are the external inbound flows a_in (D11).
#include "forest.cuh"

namespace fa {

namespace {

__device__ __forceinline__ int64_t tile_of_slot(const int64_t* __restrict__ tbase, int64_t ntiles, int64_t s) {
  int64_t lo = 0, hi = ntiles - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) / 2;
    if (tbase[mid] <= s) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// nn_dev (optional): the node count in device memory (the sync-free path;
// nn is then only the bound the grid was sized for)
__global__ void k_g1_parent(uint32_t nn, const uint32_t* __restrict__ tgt,
                            const uint8_t* __restrict__ flags, const uint32_t* __restrict__ slot_root,
                            bool cut, uint32_t* parent, const uint32_t* __restrict__ nn_dev) {
  if (nn_dev) nn = *nn_dev;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nn; v += gridDim.x * blockDim.x) {
    const uint32_t t = tgt[v];
    uint32_t p = kNone;
    if (t != kNone && !(cut && (flags[v] & NF_OUT_TILE))) p = slot_root[t];
    FA_CHECK(p == kNone || p < nn);  // a parent is a node of the same graph
    parent[v] = p;
  }
}

// x at block entry cells from the finished block exits (intra_tile: only
// edges inside a tile; cross-tile flow then arrives through x_T)
template <class T>
__global__ void k_scatter_x(uint32_t nn, const uint32_t* __restrict__ tgt, const uint8_t* __restrict__ flags,
                            const T* __restrict__ S, T* x_slot, bool intra_tile, const uint32_t* __restrict__ nn_dev) {
  if (nn_dev) nn = *nn_dev;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nn; v += gridDim.x * blockDim.x) {
    const uint32_t t = tgt[v];
    if (t != kNone && !(intra_tile && (flags[v] & NF_OUT_TILE))) atomic_add(&x_slot[t], S[v]);
  }
}

// Leaf exits (no inflow from upstream blocks) are not graph nodes: pass 1
// added their final value straight into the offset of their target slot.
// Fold those offsets into the graph value of the node the entry drains to,
// so the node's subtree sum includes them (P:L215-222 with the leaves
// raked in pass 1).
template <class T>
__global__ void k_fold_leaves(int64_t nslots, const T* __restrict__ x_slot, const uint32_t* __restrict__ slot_root,
                              T* S) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslots;
       s += (int64_t)gridDim.x * blockDim.x) {
    const T x = x_slot[s];
    if (x == (T)0) continue;
    const uint32_t e = slot_root[s];
    if (e != kNone) atomic_add(&S[e], x);  // kNone: the entry's path ends in-block (NoFlow / NoData)
  }
}

// A_T at every root of a tile-cut block-exit forest without solving it: the
// root's subtree sum is the sum of the own values (node value + folded
// leaves) of every node whose root it is (linearity), weighted by
// the product of edge weights up to the root with absorption (ptroot)
// Big trees put thousands of nodes on one root (node ids are allocated block
// by block, so neighbouring ids share roots): lanes of a warp with the same
// root are summed with shuffles first, one reduction per root per warp.
template <class T>
__global__ void k_root_sum(uint32_t nn, const uint32_t* __restrict__ troot, const T* __restrict__ own,
                           const double* __restrict__ ptroot, T* R) {
  const uint32_t stride = gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (uint32_t base = blockIdx.x * blockDim.x; base < nn; base += stride) {
    const uint32_t v = base + threadIdx.x;  // base is warp-uniform: whole warps reach the match
    const bool ok = v < nn;
    T x = (T)0;
    uint32_t r = 0xFFFFFFFFu;
    if (ok) {
      x = own[v];
      if constexpr (std::is_same<T, double>::value) {
        if (ptroot) x *= ptroot[v];
      }
      r = troot[v];
    }
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, r);
    T sum = (T)0;
    for (unsigned m = peers; m; m &= m - 1u) sum += __shfl_sync(peers, x, __ffs(m) - 1);
    if (ok && lane == __ffs(peers) - 1 && sum != (T)0) atomic_add(&R[r], sum);
  }
}

// H4 tile perimeter records of one strip: F (direction), L (Alg. 2 link) and
// A_T (tile-local accumulation, at FlowExternal slots) per tile perimeter slot
// absorption (ABS): also tile_f per slot -- a linked slot's factor to its
// tile exit (alpha product along the in-block path, slot_f, times the
// product of block-exit edge weights up to the tile root, ptroot), a
// FlowExternal slot's own alpha (the weight of its edge into the next tile)
template <class T, bool ABS = false>
__global__ void k_tile_records(Geom g, int64_t nslots, const int64_t* __restrict__ tbase,
                               const uint8_t* __restrict__ dirs, const uint32_t* __restrict__ slot_root,
                               const uint32_t* __restrict__ troot, const uint8_t* __restrict__ flags,
                               const uint32_t* __restrict__ node_slot, const T* __restrict__ S1,
                               uint32_t* links, uint8_t* fdir, T* tile_acc, const T* __restrict__ slot_f,
                               const T* __restrict__ ptroot, const float* __restrict__ alpha, T* tile_f) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslots;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = tile_of_slot(tbase, g.TR * g.TC, s), p = s - tbase[t];
    int64_t ty0, tx0, th, tw, px, py;
    g.tile_box(t, ty0, tx0, th, tw);
    perim_xy(p, th, tw, px, py);
    const int64_t gy = ty0 + py, gx = tx0 + px;
    const uint8_t d = dirs[gy * g.W + gx];
    int ly, lx;
    const int64_t b = g.block_of(gy, gx, ly, lx);
    int64_t by0, bx0;
    int bh, bw;
    g.block_box(b, by0, bx0, bh, bw);
    const int64_t bslot = b * g.pb + perim_index(lx, ly, bh, bw);
    uint32_t L = kFlowTerminates;  // Alg. 2: NoData / NoFlow / path ends inside
    T at = (T)0;
    T tf = (T)0;
    if (d >= 1 && d <= 8) {
      const int64_t ny = py + dir_dy(d), nx = px + dir_dx(d);
      const uint32_t e = slot_root[bslot];
      if (ny < 0 || nx < 0 || ny >= th || nx >= tw) {
        L = kFlowExternal;  // "c_n is outside the tile" and c = c0 (D22)
        if (e != kNone) at = S1[e];  // the cell is its own block exit
        if (ABS) tf = (T)alpha[gy * g.W + gx];
      } else if (e != kNone) {
        const uint32_t r = troot[e];
        if (flags[r] & NF_OUT_TILE) {  // the path leaves the tile at exit r
          const uint32_t rs = node_slot[r];
          const int64_t rb = rs / g.pb, rp = rs % g.pb;
          int64_t ry0, rx0;
          int rh, rw;
          g.block_box(rb, ry0, rx0, rh, rw);
          int64_t rx, ryy;
          perim_xy(rp, rh, rw, rx, ryy);
          L = (uint32_t)perim_index(rx0 + rx - tx0, ry0 + ryy - ty0, th, tw);
          if (ABS) tf = slot_f[bslot] * ptroot[e];
        }
      }
    }
    links[s] = L;
    fdir[s] = d;
    tile_acc[s] = at;
    if (ABS) tile_f[s] = tf;
  }
}

// G2, the producer's global flow graph over every tile perimeter slot of the
// whole raster: a FlowExternal slot drains into the adjoining
// tile's perimeter cell (edges or corners) unless that is NoData or off the
// DEM; a linked slot drains into its exit; the value is A_T at FlowExternal
// slots and 0 elsewhere ("set to A = 0").
template <class T, bool ABS = false>
__global__ void k_g2_slots(Geom gg, int64_t nslots, const int64_t* __restrict__ tbase,
                           const uint32_t* __restrict__ links, const uint8_t* __restrict__ fdir,
                           const T* __restrict__ tile_acc, uint32_t* parent, T* val,
                           const T* __restrict__ tile_f, T* wv2) {
  const int64_t ntiles = gg.TR * gg.TC;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslots;
       s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t L = links[s];
    uint32_t par = kNone;
    T v = (T)0;
    if (L == kFlowExternal) {
      v = tile_acc[s];
      const int64_t t = tile_of_slot(tbase, ntiles, s), p = s - tbase[t];
      int64_t ty0, tx0, th, tw, px, py;
      gg.tile_box(t, ty0, tx0, th, tw);
      perim_xy(p, th, tw, px, py);
      const int d = fdir[s];
      const int64_t ny = ty0 + py + dir_dy(d), nx = tx0 + px + dir_dx(d);
      if (ny >= 0 && nx >= 0 && ny < gg.H && nx < gg.W) {
        const int64_t t2 = (ny / gg.TH) * gg.TC + nx / gg.TW;
        int64_t y2, x2, h2, w2;
        gg.tile_box(t2, y2, x2, h2, w2);
        const int64_t s2 = tbase[t2] + perim_index(nx - x2, ny - y2, h2, w2);
        if (fdir[s2] != kNoData) par = (uint32_t)s2;
      }
    } else if (L != kFlowTerminates) {
      const int64_t t = tile_of_slot(tbase, ntiles, s);
      par = (uint32_t)(tbase[t] + L);
    }
    parent[s] = par;
    val[s] = v;
    if (ABS) wv2[s] = par == kNone ? (T)0 : tile_f[s];  // absorption: alpha (external) or path factor (linked)
  }
}

// offsets x_T(u) = sum of S over FlowExternal slots draining into u (a_in)
template <class T, bool ABS = false>
__global__ void k_xT(int64_t nslots, const uint32_t* __restrict__ parent, const uint32_t* __restrict__ links,
                     const T* __restrict__ S2, T* xT, const T* __restrict__ tile_f) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslots;
       s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t u = parent[s];
    if (u != kNone && links[s] == kFlowExternal) atomic_add(&xT[u], ABS ? S2[s] * tile_f[s] : S2[s]);
  }
}

// inject the offsets of a strip's tile slots: into pass 2 at the entry cell,
// and into the tile-cut block-exit graph at the exit its in-block path reaches
template <class T, bool ABS = false>
__global__ void k_inject_slots(Geom g, int64_t nslots, const int64_t* __restrict__ tbase,
                               const T* __restrict__ xT, const uint32_t* __restrict__ slot_root, T* val1,
                               T* x_slot, const T* __restrict__ slot_f) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslots;
       s += (int64_t)gridDim.x * blockDim.x) {
    const T x = xT[s];
    if (x == (T)0) continue;
    const int64_t t = tile_of_slot(tbase, g.TR * g.TC, s), p = s - tbase[t];
    int64_t ty0, tx0, th, tw, px, py;
    g.tile_box(t, ty0, tx0, th, tw);
    perim_xy(p, th, tw, px, py);
    int ly, lx;
    const int64_t b = g.block_of(ty0 + py, tx0 + px, ly, lx);
    int64_t by0, bx0;
    int bh, bw;
    g.block_box(b, by0, bx0, bh, bw);
    const int64_t bslot = b * g.pb + perim_index(lx, ly, bh, bw);
    atomic_add(&x_slot[bslot], x);
    const uint32_t e = slot_root[bslot];
    if (e != kNone) atomic_add(&val1[e], ABS ? x * slot_f[bslot] : x);  // reaches the block exit scaled by f
  }
}

}  // namespace

cudaError_t launch_g1_parent(cudaStream_t st, uint32_t nn, const uint32_t* tgt, const uint8_t* flags,
                             const uint32_t* slot_root, bool cut, uint32_t* parent, const uint32_t* nn_dev) {
  k_g1_parent<<<grid_for(nn), 256, 0, st>>>(nn, tgt, flags, slot_root, cut, parent, nn_dev);
  return cudaGetLastError();
}

namespace {
template <class T>
__global__ void k_copy_n(uint32_t nmax, const uint32_t* __restrict__ n_dev, const T* __restrict__ src, T* dst) {
  const uint32_t n = *n_dev;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n && v < nmax; v += gridDim.x * blockDim.x)
    dst[v] = src[v];
}
}  // namespace

// dst[0, *n_dev) = src (the node values, with the node count on the device)
template <class T>
cudaError_t launch_copy_n(cudaStream_t st, uint32_t nmax, const uint32_t* n_dev, const T* src, T* dst) {
  k_copy_n<T><<<grid_for(nmax), 256, 0, st>>>(nmax, n_dev, src, dst);
  return cudaGetLastError();
}
template cudaError_t launch_copy_n<uint32_t>(cudaStream_t, uint32_t, const uint32_t*, const uint32_t*, uint32_t*);
template cudaError_t launch_copy_n<unsigned long long>(cudaStream_t, uint32_t, const uint32_t*,
                                                       const unsigned long long*, unsigned long long*);
template cudaError_t launch_copy_n<double>(cudaStream_t, uint32_t, const uint32_t*, const double*, double*);

#ifndef FA_FOLD_VEC
#define FA_FOLD_VEC 0  // fold: 8-byte offsets read two at a time (16-byte loads): cfg3 graph 1.565 -> 1.535 ms, parity-green; off in the profiled build
#endif
// the same fold with two 8-byte offsets per load (the scan over all slots is
// a plain stream: most offsets are zero)
template <class T>
__global__ void k_fold_leaves2(int64_t npairs, const T* __restrict__ x_slot, const uint32_t* __restrict__ slot_root,
                               T* S) {
  static_assert(sizeof(T) == 8, "pairs of 8-byte offsets");
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npairs;
       i += (int64_t)gridDim.x * blockDim.x) {
    const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(x_slot) + i);
    T x0, x1;
    memcpy(&x0, &v.x, 8);
    memcpy(&x1, &v.y, 8);
    if (x0 != (T)0) {
      const uint32_t e = slot_root[2 * i];
      if (e != kNone) atomic_add(&S[e], x0);
    }
    if (x1 != (T)0) {
      const uint32_t e = slot_root[2 * i + 1];
      if (e != kNone) atomic_add(&S[e], x1);
    }
  }
}

template <class T>
cudaError_t launch_fold_leaves(cudaStream_t st, int64_t nslots, const T* x_slot, const uint32_t* slot_root, T* S) {
#if FA_FOLD_VEC
  if constexpr (sizeof(T) == 8) {
    if ((reinterpret_cast<uintptr_t>(x_slot) & 15) == 0 && nslots >= 2) {
      const int64_t np = nslots / 2;
      k_fold_leaves2<T><<<grid_for(np), 256, 0, st>>>(np, x_slot, slot_root, S);
      if (nslots & 1) k_fold_leaves<T><<<1, 32, 0, st>>>(1, x_slot + (nslots - 1), slot_root + (nslots - 1), S);
      return cudaGetLastError();
    }
  }
#endif
  k_fold_leaves<T><<<grid_for(nslots), 256, 0, st>>>(nslots, x_slot, slot_root, S);
  return cudaGetLastError();
}
template cudaError_t launch_fold_leaves<uint32_t>(cudaStream_t, int64_t, const uint32_t*, const uint32_t*, uint32_t*);
template cudaError_t launch_fold_leaves<unsigned long long>(cudaStream_t, int64_t, const unsigned long long*,
                                                            const uint32_t*, unsigned long long*);
template cudaError_t launch_fold_leaves<double>(cudaStream_t, int64_t, const double*, const uint32_t*, double*);

template <class T>
cudaError_t launch_root_sum(cudaStream_t st, uint32_t nn, const uint32_t* troot, const T* own, const double* ptroot,
                            T* R) {
  if (nn == 0) return cudaSuccess;
  k_root_sum<T><<<grid_for(nn), 256, 0, st>>>(nn, troot, own, ptroot, R);
  return cudaGetLastError();
}
template cudaError_t launch_root_sum<uint32_t>(cudaStream_t, uint32_t, const uint32_t*, const uint32_t*,
                                               const double*, uint32_t*);
template cudaError_t launch_root_sum<unsigned long long>(cudaStream_t, uint32_t, const uint32_t*,
                                                         const unsigned long long*, const double*,
                                                         unsigned long long*);
template cudaError_t launch_root_sum<double>(cudaStream_t, uint32_t, const uint32_t*, const double*, const double*,
                                             double*);

template <class T>
cudaError_t launch_scatter_x(cudaStream_t st, uint32_t nn, const uint32_t* tgt, const uint8_t* flags,
                             const T* S, T* x_slot, bool intra_tile, const uint32_t* nn_dev) {
  k_scatter_x<T><<<grid_for(nn), 256, 0, st>>>(nn, tgt, flags, S, x_slot, intra_tile, nn_dev);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_tile_records(cudaStream_t st, const Geom& g, int64_t nslots, const int64_t* tbase,
                                const uint8_t* dirs, const uint32_t* slot_root, const uint32_t* troot,
                                const uint8_t* flags, const uint32_t* node_slot, const T* S1,
                                uint32_t* links, uint8_t* fdir, T* tile_acc, const T* slot_f, const T* ptroot,
                                const float* alpha, T* tile_f) {
  if (nslots <= 0) return cudaSuccess;
  if (tile_f)
    k_tile_records<T, true><<<grid_for(nslots), 256, 0, st>>>(g, nslots, tbase, dirs, slot_root, troot, flags,
                                                               node_slot, S1, links, fdir, tile_acc, slot_f,
                                                               ptroot, alpha, tile_f);
  else
    k_tile_records<T><<<grid_for(nslots), 256, 0, st>>>(g, nslots, tbase, dirs, slot_root, troot, flags,
                                                         node_slot, S1, links, fdir, tile_acc, nullptr, nullptr,
                                                         nullptr, nullptr);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_g2_slots(cudaStream_t st, const Geom& gg, int64_t nslots, const int64_t* tbase,
                            const uint32_t* links, const uint8_t* fdir, const T* tile_acc, uint32_t* parent,
                            T* val, const T* tile_f, T* wv2) {
  if (nslots <= 0) return cudaSuccess;
  if (tile_f)
    k_g2_slots<T, true><<<grid_for(nslots), 256, 0, st>>>(gg, nslots, tbase, links, fdir, tile_acc, parent, val,
                                                           tile_f, wv2);
  else
    k_g2_slots<T><<<grid_for(nslots), 256, 0, st>>>(gg, nslots, tbase, links, fdir, tile_acc, parent, val,
                                                     nullptr, nullptr);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_xT(cudaStream_t st, int64_t nslots, const uint32_t* parent, const uint32_t* links,
                      const T* S2, T* xT, const T* tile_f) {
  if (nslots <= 0) return cudaSuccess;
  if (tile_f) k_xT<T, true><<<grid_for(nslots), 256, 0, st>>>(nslots, parent, links, S2, xT, tile_f);
  else k_xT<T><<<grid_for(nslots), 256, 0, st>>>(nslots, parent, links, S2, xT, nullptr);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_inject_slots(cudaStream_t st, const Geom& g, int64_t nslots, const int64_t* tbase,
                                const T* xT, const uint32_t* slot_root, T* val1, T* x_slot, const T* slot_f) {
  if (nslots <= 0) return cudaSuccess;
  if (slot_f)
    k_inject_slots<T, true><<<grid_for(nslots), 256, 0, st>>>(g, nslots, tbase, xT, slot_root, val1, x_slot, slot_f);
  else
    k_inject_slots<T><<<grid_for(nslots), 256, 0, st>>>(g, nslots, tbase, xT, slot_root, val1, x_slot, nullptr);
  return cudaGetLastError();
}

#define FA_INST(T)                                                                                  \
  template cudaError_t launch_scatter_x<T>(cudaStream_t, uint32_t, const uint32_t*, const uint8_t*,  \
                                           const T*, T*, bool, const uint32_t*);                                     \
  template cudaError_t launch_tile_records<T>(cudaStream_t, const Geom&, int64_t, const int64_t*,   \
                                              const uint8_t*, const uint32_t*, const uint32_t*,     \
                                              const uint8_t*, const uint32_t*, const T*, uint32_t*, \
                                              uint8_t*, T*, const T*, const T*, const float*, T*);  \
  template cudaError_t launch_g2_slots<T>(cudaStream_t, const Geom&, int64_t, const int64_t*,       \
                                          const uint32_t*, const uint8_t*, const T*, uint32_t*, T*,  \
                                          const T*, T*);                                            \
  template cudaError_t launch_xT<T>(cudaStream_t, int64_t, const uint32_t*, const uint32_t*, const T*, \
                                    T*, const T*);                                                  \
  template cudaError_t launch_inject_slots<T>(cudaStream_t, const Geom&, int64_t, const int64_t*,   \
                                              const T*, const uint32_t*, T*, T*, const T*);
FA_INST(uint32_t)
FA_INST(unsigned long long)
FA_INST(double)
#undef FA_INST

// ---------------------------------------------------------------- absorption (N3)
// Block-exit graph with multiplicative edges: exit node v sends
// alpha(v) S(v) into its target entry slot t, and the entry's offset reaches
// the exit its path drains to scaled by f(t), the product of alpha along
// that in-block path before the exit (pass 1 records): edge weight
// alpha(v) f(t).
__global__ void k_node_weights(uint32_t nn, const float* __restrict__ node_alpha, const uint32_t* __restrict__ tgt,
                               const double* __restrict__ slot_f, double* wv) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nn; v += gridDim.x * blockDim.x) {
    const uint32_t t = tgt[v];
    wv[v] = t == kNone ? 0.0 : (double)node_alpha[v] * slot_f[t];
  }
}
// leaves' pushes (already alpha(leaf) A_B(leaf)) into the node their entry drains to
__global__ void k_fold_leaves_w(int64_t nslots, const double* __restrict__ x_slot,
                                const uint32_t* __restrict__ slot_root, const double* __restrict__ slot_f,
                                double* S) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslots;
       s += (int64_t)gridDim.x * blockDim.x) {
    const double x = x_slot[s];
    if (x == 0.0) continue;
    const uint32_t e = slot_root[s];
    if (e != kNone) atomic_add(&S[e], x * slot_f[s]);
  }
}
// offsets at entry slots from the finished exits: alpha(v) S(v)
__global__ void k_scatter_x_w(uint32_t nn, const uint32_t* __restrict__ tgt, const float* __restrict__ node_alpha,
                              const double* __restrict__ S, double* x_slot, const uint8_t* __restrict__ flags,
                              bool intra_tile) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nn; v += gridDim.x * blockDim.x) {
    const uint32_t t = tgt[v];
    if (t != kNone && !(intra_tile && (flags[v] & NF_OUT_TILE))) atomic_add(&x_slot[t], (double)node_alpha[v] * S[v]);
  }
}

cudaError_t launch_absorb_graph(cudaStream_t st, uint32_t nn, int64_t nslots, const float* node_alpha,
                                const uint32_t* tgt, const double* slot_f, const double* x_slot,
                                const uint32_t* slot_root, double* wv, double* S) {
  k_node_weights<<<grid_for(nn), 256, 0, st>>>(nn, node_alpha, tgt, slot_f, wv);
  k_fold_leaves_w<<<grid_for(nslots), 256, 0, st>>>(nslots, x_slot, slot_root, slot_f, S);
  return cudaGetLastError();
}
// tile-cut graphs: edges leaving a tile are not edges of the strip graph
__global__ void k_g1_weights_cut(uint32_t nn, const uint8_t* __restrict__ flags, double* wv) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nn; v += gridDim.x * blockDim.x)
    if (flags[v] & NF_OUT_TILE) wv[v] = 0.0;
}
cudaError_t launch_g1_weights_cut(cudaStream_t st, uint32_t nn, const uint8_t* flags, double* wv) {
  k_g1_weights_cut<<<grid_for(nn), 256, 0, st>>>(nn, flags, wv);
  return cudaGetLastError();
}
cudaError_t launch_scatter_x_absorb(cudaStream_t st, uint32_t nn, const uint32_t* tgt, const float* node_alpha,
                                    const double* S, double* x_slot, const uint8_t* flags, bool intra_tile) {
  k_scatter_x_w<<<grid_for(nn), 256, 0, st>>>(nn, tgt, node_alpha, S, x_slot, flags, intra_tile);
  return cudaGetLastError();
}

}  // namespace fa
