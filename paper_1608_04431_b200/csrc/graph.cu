// graph.cu -- block-exit graph G1, tile perimeter graph G2 and the offsets.
//
// Nodes of G1 are the block exit cells written by pass 1 (one per block
// perimeter cell whose direction leaves its block, Alg. 2 "FlowExternal" at
// block level).  parent(e) = the exit reached in the target's block by the
// target cell's in-block path (slot_root), i.e. the paper's producer graph
// ("adjoining edges (or corners)") with the entry->exit links of
// Alg. 2 composed in.  Cutting the edges that leave a paper tile gives the
// per-tile problem (Alg. 1 on the tile); the tile exits then form
// G2, the paper's global flow graph.
#include "forest.cuh"

namespace fa {

namespace {

__global__ void k_g1_parent(uint32_t nn, const uint32_t* __restrict__ tgt,
                            const uint8_t* __restrict__ flags, const uint32_t* __restrict__ slot_root,
                            bool cut, uint32_t* parent) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nn; v += gridDim.x * blockDim.x) {
    const uint32_t t = tgt[v];
    uint32_t p = kNone;
    if (t != kNone && !(cut && (flags[v] & NF_OUT_TILE))) p = slot_root[t];
    parent[v] = p;
  }
}

template <class T>
__global__ void k_scatter_x(uint32_t nn, const uint32_t* __restrict__ tgt, const T* __restrict__ S,
                            T* x_slot) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nn; v += gridDim.x * blockDim.x) {
    const uint32_t t = tgt[v];
    if (t != kNone) atomic_add(&x_slot[t], S[v]);
  }
}

// G2 over tile exits: parent = tile-level root of the entry's in-tile path
// when it is a tile exit (Alg. 2 link), else none (FlowTerminates or dead).
// Value = A_T at FlowExternal nodes, 0 otherwise ("set to A = 0").
template <class T>
__global__ void k_g2(uint32_t nn, const uint32_t* __restrict__ tgt, const uint8_t* __restrict__ flags,
                     const uint32_t* __restrict__ slot_root, const uint32_t* __restrict__ troot,
                     const T* __restrict__ S1, uint32_t* parent2, T* val2) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nn; v += gridDim.x * blockDim.x) {
    const uint8_t f = flags[v];
    uint32_t p = kNone;
    T val = (T)0;
    if (f & NF_OUT_TILE) {
      val = S1[v];
      const uint32_t t = tgt[v];
      if (t != kNone) {
        const uint32_t g = slot_root[t];
        if (g != kNone) {
          const uint32_t r = troot[g];
          if (flags[r] & NF_OUT_TILE) p = r;
        }
      }
    }
    parent2[v] = p;
    val2[v] = val;
  }
}

// inject the tile offsets x_T into G1 at the entry's block exit, and record
// x_T per block slot (the paper's A' returned to each tile, read as a_in).
template <class T>
__global__ void k_inject(uint32_t nn, const uint32_t* __restrict__ tgt, const uint8_t* __restrict__ flags,
                         const uint32_t* __restrict__ slot_root, const T* __restrict__ S2, T* val1,
                         T* xT_slot) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nn; v += gridDim.x * blockDim.x) {
    if (!(flags[v] & NF_OUT_TILE)) continue;
    const uint32_t t = tgt[v];
    if (t == kNone) continue;
    const T s = S2[v];
    if (xT_slot) atomic_add(&xT_slot[t], s);
    const uint32_t g = slot_root[t];
    if (g != kNone) atomic_add(&val1[g], s);
  }
}

// H4 tile perimeter records (links, A_T, x_T) for every tile perimeter slot
template <class T>
__global__ void k_tile_records(Geom g, int64_t nslots, const int64_t* __restrict__ tbase,
                               const uint8_t* __restrict__ dirs, const uint32_t* __restrict__ slot_root,
                               const uint32_t* __restrict__ troot, const uint8_t* __restrict__ flags,
                               const uint32_t* __restrict__ node_slot, const T* __restrict__ S1,
                               const T* __restrict__ xT_slot, uint32_t* links, T* tile_acc, T* offs) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslots;
       s += (int64_t)gridDim.x * blockDim.x) {
    // tile of slot s: binary search in tbase
    int64_t lo = 0, hi = g.TR * g.TC - 1;
    while (lo < hi) {
      int64_t mid = (lo + hi + 1) / 2;
      if (tbase[mid] <= s) lo = mid; else hi = mid - 1;
    }
    const int64_t t = lo, p = s - tbase[t];
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
    uint32_t L = kFlowTerminates;
    T at = (T)0;
    if (d >= 1 && d <= 8) {
      const int64_t ny = py + dir_dy(d), nx = px + dir_dx(d);
      if (ny < 0 || nx < 0 || ny >= th || nx >= tw) {
        L = kFlowExternal;
        const uint32_t e = slot_root[bslot];  // the cell is its own block exit
        if (e != kNone) at = S1[e];
      } else {
        const uint32_t e = slot_root[bslot];
        if (e != kNone) {
          const uint32_t r = troot[e];
          if (flags[r] & NF_OUT_TILE) {
            const uint32_t rs = node_slot[r];
            const int64_t rb = rs / g.pb, rp = rs % g.pb;
            int64_t ry0, rx0;
            int rh, rw;
            g.block_box(rb, ry0, rx0, rh, rw);
            int64_t rx, ryy;
            perim_xy(rp, rh, rw, rx, ryy);
            L = (uint32_t)perim_index(rx0 + rx - tx0, ry0 + ryy - ty0, th, tw);
          }
        }
      }
    }
    if (links) links[s] = L;
    if (tile_acc) tile_acc[s] = at;
    if (offs) offs[s] = xT_slot ? xT_slot[bslot] : (T)0;
  }
}

}  // namespace

cudaError_t launch_g1_parent(cudaStream_t st, uint32_t nn, const uint32_t* tgt, const uint8_t* flags,
                             const uint32_t* slot_root, bool cut, uint32_t* parent) {
  k_g1_parent<<<grid_for(nn), 256, 0, st>>>(nn, tgt, flags, slot_root, cut, parent);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_scatter_x(cudaStream_t st, uint32_t nn, const uint32_t* tgt, const T* S, T* x_slot) {
  k_scatter_x<T><<<grid_for(nn), 256, 0, st>>>(nn, tgt, S, x_slot);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_g2(cudaStream_t st, uint32_t nn, const uint32_t* tgt, const uint8_t* flags,
                      const uint32_t* slot_root, const uint32_t* troot, const T* S1, uint32_t* parent2,
                      T* val2) {
  k_g2<T><<<grid_for(nn), 256, 0, st>>>(nn, tgt, flags, slot_root, troot, S1, parent2, val2);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_inject(cudaStream_t st, uint32_t nn, const uint32_t* tgt, const uint8_t* flags,
                          const uint32_t* slot_root, const T* S2, T* val1, T* xT_slot) {
  k_inject<T><<<grid_for(nn), 256, 0, st>>>(nn, tgt, flags, slot_root, S2, val1, xT_slot);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_tile_records(cudaStream_t st, const Geom& g, int64_t nslots, const int64_t* tbase,
                                const uint8_t* dirs, const uint32_t* slot_root, const uint32_t* troot,
                                const uint8_t* flags, const uint32_t* node_slot, const T* S1,
                                const T* xT_slot, uint32_t* links, T* tile_acc, T* offs) {
  k_tile_records<T><<<grid_for(nslots), 256, 0, st>>>(g, nslots, tbase, dirs, slot_root, troot, flags,
                                                       node_slot, S1, xT_slot, links, tile_acc, offs);
  return cudaGetLastError();
}

#define FA_INST(T)                                                                                 \
  template cudaError_t launch_scatter_x<T>(cudaStream_t, uint32_t, const uint32_t*, const T*, T*); \
  template cudaError_t launch_g2<T>(cudaStream_t, uint32_t, const uint32_t*, const uint8_t*,       \
                                    const uint32_t*, const uint32_t*, const T*, uint32_t*, T*);    \
  template cudaError_t launch_inject<T>(cudaStream_t, uint32_t, const uint32_t*, const uint8_t*,   \
                                        const uint32_t*, const T*, T*, T*);                        \
  template cudaError_t launch_tile_records<T>(cudaStream_t, const Geom&, int64_t, const int64_t*,  \
                                              const uint8_t*, const uint32_t*, const uint32_t*,    \
                                              const uint8_t*, const uint32_t*, const T*, const T*, \
                                              uint32_t*, T*, T*);
FA_INST(uint32_t)
FA_INST(unsigned long long)
FA_INST(double)
#undef FA_INST

}  // namespace fa
