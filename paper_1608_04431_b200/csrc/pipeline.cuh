// pipeline.cuh -- host orchestration shared by the entry points of libfa
// (api.cu: one device, out of core, absorption; dist.cu: one strip per rank):
// the context, argument staging, and the per-strip phases of the tiled method
//   phase A (per strip): pass 1 with halo rows, tile-cut block-exit graph ->
//     A_T, tile roots -> tile perimeter records (F, A, L)
//   exchange: the records of every strip reach every strip / rank
//   phase B (per strip): the producer's global graph over all tile perimeter
//     slots, solved redundantly -> offsets x_T (a_in, D11) ->
//     injected into the strip's tile-cut graph -> finalize (RETAIN P:L260 /
//     EVICT P:L255-262).
// Internal to libfa (included by api.cu and dist.cu only).
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "fa.h"
#include "forest.cuh"
#include "nccl.h"

namespace fa {

template <class T, int WK>
cudaError_t launch_pass1(const PassArgs<T, WK>& a, bool from_dem, cudaStream_t st);
template <class T, int WK>
cudaError_t launch_pass2(const PassArgs<T, WK>& a, cudaStream_t st);
template <class T>
cudaError_t launch_retain(const Geom& g, const T* x_slot, const uint8_t* dirs, T* acc, cudaStream_t st,
                          int64_t bbeg = 0, int64_t bend = -1);
cudaError_t launch_d8(const float* dem, const float* dem_up, const float* dem_dn, int64_t H, int64_t W,
                      float nodata, uint8_t* dirs,
                      cudaStream_t st);
cudaError_t launch_g1_parent(cudaStream_t st, uint32_t nn, const uint32_t* tgt, const uint8_t* flags,
                             const uint32_t* slot_root, bool cut, uint32_t* parent,
                             const uint32_t* nn_dev = nullptr);
template <class T>
cudaError_t launch_copy_n(cudaStream_t st, uint32_t nmax, const uint32_t* n_dev, const T* src, T* dst);
// absorption: block.cu / graph.cu
cudaError_t launch_pass1_absorb(const PassArgs<double, 0>* a0, const PassArgs<double, 2>* a2, bool from_dem,
                                cudaStream_t st);
cudaError_t launch_retain_absorb(const Geom& g, const double* x_slot, const uint8_t* dirs, double* acc,
                                 const float* alpha, cudaStream_t st);
cudaError_t launch_absorb_graph(cudaStream_t st, uint32_t nn, int64_t nslots, const float* node_alpha,
                                const uint32_t* tgt, const double* slot_f, const double* x_slot,
                                const uint32_t* slot_root, double* wv, double* S);
cudaError_t launch_scatter_x_absorb(cudaStream_t st, uint32_t nn, const uint32_t* tgt, const float* node_alpha,
                                    const double* S, double* x_slot, const uint8_t* flags, bool intra_tile);
cudaError_t launch_g1_weights_cut(cudaStream_t st, uint32_t nn, const uint8_t* flags, double* wv);
// depression filling (N4): fill.cu
cudaError_t fill_depressions(Runtime& rt, const float* z, int64_t H, int64_t W, float nodata, float* out, int tile);
template <class T>
cudaError_t launch_scatter_x(cudaStream_t st, uint32_t nn, const uint32_t* tgt, const uint8_t* flags,
                             const T* S, T* x_slot, bool intra_tile, const uint32_t* nn_dev = nullptr);
template <class T>
cudaError_t launch_fold_leaves(cudaStream_t st, int64_t nslots, const T* x_slot, const uint32_t* slot_root, T* S);
template <class T>
cudaError_t launch_root_sum(cudaStream_t st, uint32_t nn, const uint32_t* troot, const T* own, const double* ptroot,
                            T* R);
template <class T>
cudaError_t launch_tile_records(cudaStream_t st, const Geom& g, int64_t nslots, const int64_t* tbase,
                                const uint8_t* dirs, const uint32_t* slot_root, const uint32_t* troot,
                                const uint8_t* flags, const uint32_t* node_slot, const T* S1,
                                uint32_t* links, uint8_t* fdir, T* tile_acc, const T* slot_f = nullptr,
                                const T* ptroot = nullptr, const float* alpha = nullptr, T* tile_f = nullptr);
template <class T>
cudaError_t launch_g2_slots(cudaStream_t st, const Geom& gg, int64_t nslots, const int64_t* tbase,
                            const uint32_t* links, const uint8_t* fdir, const T* tile_acc, uint32_t* parent,
                            T* val, const T* tile_f = nullptr, T* wv2 = nullptr);
template <class T>
cudaError_t launch_xT(cudaStream_t st, int64_t nslots, const uint32_t* parent, const uint32_t* links,
                      const T* S2, T* xT, const T* tile_f = nullptr);
template <class T>
cudaError_t launch_inject_slots(cudaStream_t st, const Geom& g, int64_t nslots, const int64_t* tbase,
                                const T* xT, const uint32_t* slot_root, T* val1, T* x_slot,
                                const T* slot_f = nullptr);

// ---------------------------------------------------------------- NCCL (dlopen)
struct Nccl {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
  bool load() {
    if (h) return true;
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
#define FA_SYM(f, n) f = reinterpret_cast<decltype(f)>(dlsym(h, n))
    FA_SYM(getUniqueId, "ncclGetUniqueId");
    FA_SYM(commInitRank, "ncclCommInitRank");
    FA_SYM(commDestroy, "ncclCommDestroy");
    FA_SYM(groupStart, "ncclGroupStart");
    FA_SYM(groupEnd, "ncclGroupEnd");
    FA_SYM(send, "ncclSend");
    FA_SYM(recv, "ncclRecv");
    FA_SYM(broadcast, "ncclBroadcast");
    FA_SYM(allReduce, "ncclAllReduce");
    FA_SYM(allGather, "ncclAllGather");
    FA_SYM(errorString, "ncclGetErrorString");
#undef FA_SYM
    return getUniqueId && commInitRank && commDestroy && groupStart && groupEnd && send && recv &&
           broadcast && allReduce && allGather && errorString;
  }
};
inline Nccl& nccl() {
  static Nccl n;
  return n;
}

Geom make_geom(int64_t H, int64_t W, int64_t th, int64_t tw, int br);


}  // namespace fa

struct fa_ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  int64_t tile_r = 0, tile_c = 0;
  std::string err;
  fa::Runtime rt;
  fa_stats stats{};
  cudaEvent_t ev[10]{};  // [0..3] phases, [4..6] D8 / block kernel, [8..9] multi-GPU exchange
  uint32_t* d_small = nullptr;  // [0]=node_count [1]=status [2..3]=wsum(u64) [4..15] scratch
  uint32_t* h_small = nullptr;
  // out-of-core streaming (fa_accumulate_streamed): copy stream + buffer events
  cudaStream_t cs = nullptr, cs_out = nullptr;  // uploads / downloads (PCIe is full duplex)
  cudaEvent_t ev_in[2]{}, ev_used[2]{}, ev_out[2]{};
  // multi-GPU
  ncclComm_t comm = nullptr;
  int rank = -1, nranks = 0;
  unsigned char comm_id[128]{};
  // options (fa_set_option): the paper's memory retention strategy,
  // D8 split or fused into pass 1, block rows, graph walk cap, fill tile
  int opt_evict = 0;
  int opt_fused = 0;
  int opt_br = fa::kBR;
  int opt_walk_cap = 128;
  int opt_fill_tile = 32;
  int opt_values = FA_VALUES_L2;
  int opt_graph = FA_GRAPH_AUTO;
  int opt_dist_records = FA_DIST_STRIPS;
  bool no_sync_free = false;  // set while a small-raster call reruns host-driven
  bool retain() const { return opt_evict == 0; }
};

namespace {

using fa::Geom;

fa_status set_err(fa_ctx* c, fa_status s, const std::string& m) {
  if (c) c->err = m;
  return s;
}

#define CK(...)                                                                         \
  do {                                                                                  \
    cudaError_t _e = (__VA_ARGS__);                                                     \
    if (_e != cudaSuccess)                                                              \
      return set_err(ctx, FA_E_CUDA, std::string(#__VA_ARGS__ " failed: ") + cudaGetErrorString(_e)); \
  } while (0)

#define NK(...)                                                                         \
  do {                                                                                  \
    ncclResult_t _r = (__VA_ARGS__);                                                    \
    if (_r != ncclSuccess)                                                              \
      return set_err(ctx, FA_E_NCCL, std::string(#__VA_ARGS__ " failed: ") + fa::nccl().errorString(_r)); \
  } while (0)

#define FS(...)                        \
  do {                                 \
    fa_status _s = (__VA_ARGS__);      \
    if (_s != FA_OK) return _s;        \
  } while (0)

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// host buffers are staged through device memory (stream-ordered)
struct Staged {
  void* dev = nullptr;
  bool owned = false;
};
cudaError_t stage_in(cudaStream_t st, const void* p, size_t bytes, Staged& s) {
  if (!p) return cudaSuccess;
  if (is_device_ptr(p)) {
    s.dev = const_cast<void*>(p);
    return cudaSuccess;
  }
  cudaError_t e = cudaMallocAsync(&s.dev, bytes, st);
  if (e) return e;
  s.owned = true;
  return cudaMemcpyAsync(s.dev, p, bytes, cudaMemcpyHostToDevice, st);
}
cudaError_t stage_out_alloc(cudaStream_t st, void* p, size_t bytes, Staged& s) {
  if (!p) return cudaSuccess;
  if (is_device_ptr(p)) {
    s.dev = p;
    return cudaSuccess;
  }
  s.owned = true;
  return cudaMallocAsync(&s.dev, bytes, st);
}

int64_t tile_perim_total(const Geom& g, std::vector<int64_t>* base) {
  int64_t tot = 0;
  if (base) base->assign(g.TR * g.TC + 1, 0);
  for (int64_t t = 0; t < g.TR * g.TC; ++t) {
    int64_t y0, x0, h, w;
    g.tile_box(t, y0, x0, h, w);
    if (base) (*base)[t] = tot;
    tot += fa::perim_count(h, w);
  }
  if (base) (*base)[g.TR * g.TC] = tot;
  return tot;
}

// ---------------------------------------------------------------- strip state
template <class T>
struct Strip {
  Geom g{};               // strip geometry (H = strip rows; tiling as configured)
  int64_t row_begin = 0;  // global row of strip row 0
  const float* dem = nullptr;
  const float* dem_up = nullptr;
  const float* dem_dn = nullptr;
  const float* dem_up2 = nullptr;  // rows -2 / H+1 (null: off-grid) when halo2: the D8 of the halo rows
  const float* dem_dn2 = nullptr;
  bool halo2 = false;
  const uint8_t* dirs = nullptr;
  const uint8_t* dirs_up = nullptr;
  const uint8_t* dirs_dn = nullptr;
  const void* w = nullptr;
  T* acc = nullptr;
  float nodata = 0;
  // device state
  T* acc_tmp = nullptr;   // in-place accumulation buffer when the caller wants no raster
  uint8_t* halo_dirs = nullptr;  // D8 codes of rows -1 and H (split path, strips)
  const float* alpha = nullptr;  // absorption (N3): per-cell alpha, or null
  T* slot_f = nullptr;           // absorption: alpha product along each entry slot's path
  float* node_alpha = nullptr;   // absorption: alpha at each node's exit cell
  double* wv = nullptr;          // absorption: block-exit edge weights (tile-cut graph)
  double* ptroot = nullptr;      // absorption: edge-weight product from each node to its tile root
  uint8_t* dirs_buf = nullptr;
  uint32_t* slot_root = nullptr;
  T* node_val = nullptr;
  uint32_t* node_slot = nullptr;
  uint32_t* node_tgt = nullptr;
  uint8_t* node_flags = nullptr;
  T* x_slot = nullptr;
  uint32_t nn = 0;
  uint32_t* parent = nullptr;
  T* S = nullptr;
  uint32_t* troot = nullptr;
  int64_t slot0 = 0, nslots = 0;  // this strip's range of global tile perimeter slots
  int64_t* dtbase = nullptr;      // local tile slot bases (device)
  bool own_in_S = false;          // S holds node values + folded leaves (strip_records): phase B starts there
  void release(fa::Runtime& rt) {
    for (void* p : {(void*)dirs_buf, (void*)slot_root, (void*)node_val, (void*)node_slot, (void*)node_tgt,
                    (void*)node_flags, (void*)x_slot, (void*)parent, (void*)S, (void*)troot, (void*)dtbase,
                    (void*)acc_tmp, (void*)halo_dirs, (void*)slot_f, (void*)node_alpha, (void*)wv,
                    (void*)ptroot})
      rt.free(p);
    wv = ptroot = nullptr;
    dirs_buf = nullptr;
    acc_tmp = nullptr;
    halo_dirs = nullptr;
    slot_f = nullptr;
    node_alpha = nullptr;
    slot_root = node_slot = node_tgt = parent = troot = nullptr;
    node_val = x_slot = S = nullptr;
    node_flags = nullptr;
    dtbase = nullptr;
  }
  const uint8_t* dirs_in() const { return dem ? dirs_buf : dirs; }
};

template <class T, int WK>
fa::PassArgs<T, WK> pass_args(fa_ctx* ctx, Strip<T>& s) {
  fa::PassArgs<T, WK> a{};
  a.g = s.g;
  a.dem = s.dem;
  a.nodata = s.nodata;
  a.dirs_in = s.dirs_in();
  a.dirs_out = s.dirs_buf;
  a.w = s.w;
  a.dem_up = s.dem_up;
  a.dem_dn = s.dem_dn;
  a.dirs_up = s.dirs_up;
  a.dirs_dn = s.dirs_dn;
  a.node_count = ctx->d_small + 0;
  a.status = ctx->d_small + 1;
  a.wsum = reinterpret_cast<unsigned long long*>(ctx->d_small + 2);
  a.node_val = s.node_val;
  a.node_slot = s.node_slot;
  a.node_tgt = s.node_tgt;
  a.node_flags = s.node_flags;
  a.slot_root = s.slot_root;
  a.x_slot = s.x_slot;
  a.acc = s.acc ? s.acc : s.acc_tmp;  // pass 1 accumulates in place (RETAIN)
  a.retain = s.acc != nullptr && ctx->retain();
  a.vsmem = ctx->opt_values == FA_VALUES_SMEM;
  a.b_begin = 0;
  a.b_end = s.g.nblocks;
  return a;
}

// status word -> ABI status (data-dependent errors)
fa_status check_status(fa_ctx* ctx, uint32_t stat, unsigned long long wsum, bool is_u32) {
  using namespace fa;
  if (stat & ST_BADCODE) return set_err(ctx, FA_E_DIRCODE, "direction raster holds a byte outside {0..8,255}");
  if (stat & ST_BADWEIGHT) return set_err(ctx, FA_E_ARG, "f32 weights must be finite and >= 0");
  if (stat & ST_BADALPHA) return set_err(ctx, FA_E_ARG, "alpha must be a finite value in [0, 1] at data cells");
  if (is_u32 && wsum >= 0xFFFFFFFFull)
    return set_err(ctx, FA_E_OVERFLOW, "sum of weights reaches the u32 range (NoData marker); use u64");
  if (stat & ST_CYCLE) return set_err(ctx, FA_E_CYCLE, "direction graph has a cycle (some cells never retire)");
  return FA_OK;
}

// pass 1 of a strip + block-exit graph parents (cut at tile edges when `cut`)
// sync_free: the node count stays on the device (d_small[0]); parent / S are
// sized for every block slot and the kernels after pass 1 read the count
// themselves (the small-raster path of run_acc: no host round trip)
template <class T, int WK>
fa_status strip_pass1(fa_ctx* ctx, Strip<T>& s, bool cut, bool sync_free = false) {
  using namespace fa;
  cudaStream_t st = ctx->st;
  Runtime& rt = ctx->rt;
  const Geom& g = s.g;
  const int64_t slots = g.nblocks * g.pb;
  if (slots >= (int64_t)0xFFFFFFF0ll)
    return set_err(ctx, FA_E_ARG, "raster too large for one device (block slots exceed 2^32)");
  if (s.dem) s.dirs_buf = rt.alloc<uint8_t>((size_t)(g.H * g.W));
  if (!s.acc) s.acc_tmp = rt.alloc<T>((size_t)(g.H * g.W));
  s.slot_root = rt.alloc<uint32_t>(slots);
  s.node_val = rt.alloc<T>(slots);
  s.node_slot = rt.alloc<uint32_t>(slots);
  s.node_tgt = rt.alloc<uint32_t>(slots);
  s.node_flags = rt.alloc<uint8_t>(slots);
  s.x_slot = rt.alloc<T>(slots);
  if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
  CK(cudaMemsetAsync(ctx->d_small, 0, sizeof(uint32_t), st));  // node counter (status accumulates)
  CK(cudaMemsetAsync(s.x_slot, 0, slots * sizeof(T), st));
  fa::PassArgs<T, WK> pa = pass_args<T, WK>(ctx, s);
  pa.cut = cut;
  // H1 runs as its own kernel (high occupancy), then pass 1 starts from the
  // directions.  A strip also computes the codes of its halo rows -1 and H
  // (from the 2-row z halo), so pass 1 sees the neighbour strips' codes on
  // its ring.  FA_OPT_D8 = FA_D8_FUSED (or 1-row halos) keeps D8 fused into pass 1.
  const bool split = s.dem && !ctx->opt_fused && (s.halo2 || (!s.dem_up && !s.dem_dn));
  CK(cudaEventRecord(ctx->ev[4], st));
  if (split) {
    CK(launch_d8(s.dem, s.dem_up, s.dem_dn, g.H, g.W, s.nodata, s.dirs_buf, st));
    ++rt.launches;
    pa.dirs_out = nullptr;
    if (s.dem_up || s.dem_dn) {
      s.halo_dirs = rt.alloc<uint8_t>((size_t)(2 * g.W));
      if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
    }
    if (s.dem_up) {
      CK(launch_d8(s.dem_up, s.dem_up2, s.dem, 1, g.W, s.nodata, s.halo_dirs, st));
      ++rt.launches;
    }
    if (s.dem_dn) {
      CK(launch_d8(s.dem_dn, s.dem + (g.H - 1) * g.W, s.dem_dn2, 1, g.W, s.nodata, s.halo_dirs + g.W, st));
      ++rt.launches;
    }
    pa.dirs_up = s.dem_up ? s.halo_dirs : nullptr;
    pa.dirs_dn = s.dem_dn ? s.halo_dirs + g.W : nullptr;
  }
  CK(cudaEventRecord(ctx->ev[5], st));
  if (s.alpha) {
    if constexpr (std::is_same<T, double>::value && (WK == 0 || WK == 2)) {
      s.slot_f = rt.alloc<T>(slots);
      s.node_alpha = rt.alloc<float>(slots);
      if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
      pa.alpha = s.alpha;
      pa.slot_f = s.slot_f;
      pa.node_alpha = s.node_alpha;
      if constexpr (WK == 0) CK(launch_pass1_absorb(&pa, nullptr, s.dem != nullptr && !split, st));
      else CK(launch_pass1_absorb(nullptr, &pa, s.dem != nullptr && !split, st));
    } else {
      return set_err(ctx, FA_E_ARG, "absorption needs f64 output and f32 or no weights");
    }
  } else {
    CK(launch_pass1<T, WK>(pa, s.dem != nullptr && !split, st));
  }
  CK(cudaEventRecord(ctx->ev[6], st));
  ++rt.launches;
  if (sync_free) {
    s.nn = (uint32_t)slots;  // a bound: the count is ctx->d_small[0]
    s.parent = rt.alloc<uint32_t>(s.nn);
    s.S = rt.alloc<T>(s.nn);
    if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
    CK(launch_g1_parent(st, s.nn, s.node_tgt, s.node_flags, s.slot_root, cut, s.parent, ctx->d_small));
    ++rt.launches;
    return FA_OK;
  }
  CK(rt.read(ctx->d_small, 4));
  s.nn = rt.h_cnt[0];
  s.parent = rt.alloc<uint32_t>(s.nn);
  s.S = rt.alloc<T>(s.nn);
  if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
  CK(launch_g1_parent(st, s.nn, s.node_tgt, s.node_flags, s.slot_root, cut, s.parent));
  ++rt.launches;
  return FA_OK;
}

// local tile slot bases of a strip (prefix sums of the tiles' perimeter
// counts), computed on the device so no host buffer has to outlive a copy
static __global__ void k_tile_bases(fa::Geom g, int64_t* base) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  int64_t tot = 0;
  for (int64_t t = 0; t < g.TR * g.TC; ++t) {
    int64_t y0, x0, h, w;
    g.tile_box(t, y0, x0, h, w);
    base[t] = tot;
    tot += fa::perim_count(h, w);
  }
  base[g.TR * g.TC] = tot;
}

// phase A tail: A_T at block exits, tile roots, tile perimeter records; the
// output pointers are the strip's own first slot (its nslots records follow)
// parts of strip_records: everything, or the steps before / after the tile
// roots (strips rooted together as one forest: roots_strips)
enum : int { REC_ALL = 0, REC_PRE = 1, REC_POST = 2 };

template <class T>
fa_status strip_records(fa_ctx* ctx, Strip<T>& s, uint32_t* links, uint8_t* fdir, T* tile_acc,
                        T* tile_f = nullptr, int part = REC_ALL) {
  using namespace fa;
  cudaStream_t st = ctx->st;
  Runtime& rt = ctx->rt;
  if (part == REC_POST) goto post;
  s.troot = rt.alloc<uint32_t>(s.nn);
  s.nslots = tile_perim_total(s.g, nullptr);
  s.dtbase = rt.alloc<int64_t>((size_t)(s.g.TR * s.g.TC + 1));
  if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
  k_tile_bases<<<1, 32, 0, st>>>(s.g, s.dtbase);
  ++rt.launches;
  CK(cudaMemcpyAsync(s.S, s.node_val, s.nn * sizeof(T), cudaMemcpyDeviceToDevice, st));
  if constexpr (std::is_same<T, double>::value) {
    if (s.alpha) {
      // absorption: weighted tile-cut graph; tile records carry the path factors
      s.wv = rt.alloc<double>(s.nn ? s.nn : 1);
      s.ptroot = rt.alloc<double>(s.nn ? s.nn : 1);
      if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
      CK(launch_absorb_graph(st, s.nn, s.g.nblocks * s.g.pb, s.node_alpha, s.node_tgt, s.slot_f, s.x_slot,
                             s.slot_root, s.wv, s.S));
      CK(launch_g1_weights_cut(st, s.nn, s.node_flags, s.wv));
      rt.launches += 3;
      CK(forest_roots_weighted(rt, s.nn, s.parent, s.wv, s.troot, s.ptroot));
      T* R = rt.alloc<T>(s.nn);
      if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
      CK(cudaMemsetAsync(R, 0, (s.nn ? s.nn : 1) * sizeof(T), st));
      CK(launch_root_sum<T>(st, s.nn, s.troot, s.S, s.ptroot, R));
      CK(launch_tile_records<T>(st, s.g, s.nslots, s.dtbase, s.dirs_in(), s.slot_root, s.troot, s.node_flags,
                                s.node_slot, R, links, fdir, tile_acc, s.slot_f,
                                s.ptroot, s.alpha, tile_f));
      rt.launches += 2;
      rt.free(R);
      return FA_OK;
    }
  }
  CK(launch_fold_leaves<T>(st, s.g.nblocks * s.g.pb, s.x_slot, s.slot_root, s.S));  // leaves raked in pass 1
  ++rt.launches;
  if (part == REC_PRE) return FA_OK;
  // A_T is needed at the tile exits only (the roots of the tile-cut forest):
  // root ids by pointer jumping, then one reduction of the own values by
  // root -- no forest solve here; phase B (strip_finish) solves the strip
  // graph once, with the injected offsets
  CK(forest_roots(rt, s.nn, s.parent, s.troot));
post:
  {
    T* R = rt.alloc<T>(s.nn);
    if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
    CK(cudaMemsetAsync(R, 0, (s.nn ? s.nn : 1) * sizeof(T), st));
    CK(launch_root_sum<T>(st, s.nn, s.troot, s.S, nullptr, R));
    CK(launch_tile_records<T>(st, s.g, s.nslots, s.dtbase, s.dirs_in(), s.slot_root, s.troot, s.node_flags,
                              s.node_slot, R, links, fdir, tile_acc));
    rt.launches += 2;
    rt.free(R);
  }
  s.own_in_S = true;
  return FA_OK;
}

// the producer's global graph over all tile slots -> offsets x_T (all slots)
template <class T>
fa_status solve_g2(fa_ctx* ctx, const Geom& gg, int64_t nslots, const std::vector<int64_t>& hbase,
                   const uint32_t* links, const uint8_t* fdir, const T* tile_acc, T* xT,
                   const T* tile_f = nullptr) {
  using namespace fa;
  cudaStream_t st = ctx->st;
  Runtime& rt = ctx->rt;
  if (nslots >= (int64_t)0xFFFFFFF0ll) return set_err(ctx, FA_E_ARG, "too many tile perimeter slots");
  int64_t* db = rt.alloc<int64_t>(hbase.size());
  uint32_t* par = rt.alloc<uint32_t>(nslots);
  T* val = rt.alloc<T>(nslots);
  if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
  CK(cudaMemcpyAsync(db, hbase.data(), hbase.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  T* wv2 = tile_f ? rt.alloc<T>(nslots) : nullptr;
  if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
  CK(launch_g2_slots<T>(st, gg, nslots, db, links, fdir, tile_acc, par, val, tile_f, wv2));
  ++rt.launches;
  if constexpr (std::is_same<T, double>::value) {
    if (tile_f) CK(forest_solve_weighted(rt, (uint32_t)nslots, par, wv2, val));  // absorption: weighted G2
    else CK(forest_solve<T>(rt, (uint32_t)nslots, par, val));
  } else {
    CK(forest_solve<T>(rt, (uint32_t)nslots, par, val));
  }
  CK(cudaMemsetAsync(xT, 0, nslots * sizeof(T), st));
  CK(launch_xT<T>(st, nslots, par, links, val, xT, tile_f));
  ++rt.launches;
  CK(cudaStreamSynchronize(st));
  rt.free(db);
  rt.free(wv2);
  rt.free(par);
  rt.free(val);
  return FA_OK;
}

// phase B tail: inject x_T, solve the tile-cut graph, scatter, pass 2
// parts of strip_finish: everything, or the steps before / after the
// tile-cut graph solve (strips solved together as one forest: solve_strips)
enum : int { FIN_ALL = 0, FIN_PRE = 1, FIN_POST = 2 };

template <class T, int WK>
fa_status strip_finish(fa_ctx* ctx, Strip<T>& s, const T* xT_global, int part = FIN_ALL) {
  using namespace fa;
  cudaStream_t st = ctx->st;
  Runtime& rt = ctx->rt;
  if (part == FIN_POST) {
    CK(launch_scatter_x<T>(st, s.nn, s.node_tgt, s.node_flags, s.S, s.x_slot, true));
    ++rt.launches;
    if (s.acc) {
      if (ctx->retain()) CK(launch_retain<T>(s.g, s.x_slot, s.dirs_in(), s.acc, st));
      else CK(launch_pass2<T, WK>(pass_args<T, WK>(ctx, s), st));
      ++rt.launches;
    }
    return FA_OK;
  }
  if (!s.own_in_S) CK(cudaMemcpyAsync(s.S, s.node_val, s.nn * sizeof(T), cudaMemcpyDeviceToDevice, st));
  if constexpr (std::is_same<T, double>::value) {
    if (s.alpha) {
      // absorption: weighted fold, injection scaled by the entry path factor,
      // weighted tile-cut solve, weighted intra-tile scatter, alpha finalize
      if (!s.wv) {
        s.wv = rt.alloc<double>(s.nn ? s.nn : 1);
        if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
      }
      CK(launch_absorb_graph(st, s.nn, s.g.nblocks * s.g.pb, s.node_alpha, s.node_tgt, s.slot_f, s.x_slot,
                             s.slot_root, s.wv, s.S));
      CK(launch_g1_weights_cut(st, s.nn, s.node_flags, s.wv));
      rt.launches += 3;
      CK(launch_inject_slots<T>(st, s.g, s.nslots, s.dtbase, xT_global + s.slot0, s.slot_root, s.S, s.x_slot,
                                s.slot_f));
      ++rt.launches;
      CK(forest_solve_weighted(rt, s.nn, s.parent, s.wv, s.S));
      CK(launch_scatter_x_absorb(st, s.nn, s.node_tgt, s.node_alpha, s.S, s.x_slot, s.node_flags, true));
      ++rt.launches;
      if (s.acc) {
        CK(launch_retain_absorb(s.g, s.x_slot, s.dirs_in(), s.acc, s.alpha, st));
        ++rt.launches;
      }
      return FA_OK;
    }
  }
  // leaves first (x_slot holds only their pass-1 values here; strip_records
  // of the same strip object has folded them already), then x_T
  if (!s.own_in_S) {
    CK(launch_fold_leaves<T>(st, s.g.nblocks * s.g.pb, s.x_slot, s.slot_root, s.S));
    ++rt.launches;
  }
  CK(launch_inject_slots<T>(st, s.g, s.nslots, s.dtbase, xT_global + s.slot0, s.slot_root, s.S, s.x_slot));
  ++rt.launches;
  if (part == FIN_PRE) return FA_OK;
  CK(forest_solve<T>(rt, s.nn, s.parent, s.S));  // true A at every block exit
  CK(launch_scatter_x<T>(st, s.nn, s.node_tgt, s.node_flags, s.S, s.x_slot, true));
  ++rt.launches;
  if (s.acc) {
    if (ctx->retain()) CK(launch_retain<T>(s.g, s.x_slot, s.dirs_in(), s.acc, st));
    else CK(launch_pass2<T, WK>(pass_args<T, WK>(ctx, s), st));
    ++rt.launches;
  }
  return FA_OK;
}

static __global__ void k_offset_parents(uint32_t n, const uint32_t* __restrict__ par, uint32_t off,
                                        uint32_t* __restrict__ out) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint32_t p = par[v];
    out[v] = p == fa::kNone ? fa::kNone : p + off;
  }
}

// phase B on one device: the strips' tile-cut graphs are disjoint forests, so
// they are solved as ONE forest (node ids offset by strip) -- one solve and
// its handful of host reads instead of one per strip.  Returns false (nothing
// done) when the joint node count would not fit 32-bit ids.
static __global__ void k_unoffset(uint32_t n, const uint32_t* __restrict__ in, uint32_t off, uint32_t* __restrict__ out) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) out[v] = in[v] - off;
}

// the strips' tile-cut graphs are disjoint forests: their parents with node
// ids offset by strip form ONE forest (nullptr when the joint node count does
// not fit 32-bit ids); *n_out = its node count
template <class T>
uint32_t* joint_parents(fa_ctx* ctx, std::vector<Strip<T>>& strips, uint32_t* n_out) {
  using namespace fa;
  Runtime& rt = ctx->rt;
  uint64_t n = 0;
  for (auto& s : strips) n += s.nn;
  *n_out = 0;
  if (n == 0 || n >= (uint64_t)kNone) return nullptr;
  uint32_t* par = rt.alloc<uint32_t>(n);
  if (rt.err) return nullptr;
  uint32_t off = 0;
  for (auto& s : strips) {
    if (s.nn) {
      k_offset_parents<<<grid_for(s.nn), 256, 0, ctx->st>>>(s.nn, s.parent, off, par + off);
      ++rt.launches;
    }
    off += s.nn;
  }
  *n_out = (uint32_t)n;
  return par;
}

// phase A on one device: the tile roots of every strip by ONE pointer-jumping
// solve over the joint forest (roots of strip i lie in strip i: ids minus its offset)
template <class T>
fa_status roots_strips(fa_ctx* ctx, std::vector<Strip<T>>& strips, const uint32_t* par, uint32_t n) {
  using namespace fa;
  cudaStream_t st = ctx->st;
  Runtime& rt = ctx->rt;
  uint32_t* root = rt.alloc<uint32_t>(n);
  if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
  CK(forest_roots(rt, n, par, root));
  uint32_t off = 0;
  for (auto& s : strips) {
    if (s.nn) {
      k_unoffset<<<grid_for(s.nn), 256, 0, st>>>(s.nn, root + off, off, s.troot);
      ++rt.launches;
    }
    off += s.nn;
  }
  rt.free(root);
  return FA_OK;
}

// phase B on one device: the strips' tile-cut graphs solved as ONE forest --
// one solve and its handful of host reads instead of one per strip
template <class T>
fa_status solve_strips(fa_ctx* ctx, std::vector<Strip<T>>& strips, const uint32_t* par, uint32_t n) {
  using namespace fa;
  cudaStream_t st = ctx->st;
  Runtime& rt = ctx->rt;
  T* val = rt.alloc<T>(n);
  if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
  uint32_t off = 0;
  for (auto& s : strips) {
    if (s.nn) CK(cudaMemcpyAsync(val + off, s.S, s.nn * sizeof(T), cudaMemcpyDeviceToDevice, st));
    off += s.nn;
  }
  CK(forest_solve<T>(rt, n, par, val));  // true A at every block exit of every strip
  off = 0;
  for (auto& s : strips) {
    if (s.nn) CK(cudaMemcpyAsync(s.S, val + off, s.nn * sizeof(T), cudaMemcpyDeviceToDevice, st));
    off += s.nn;
  }
  rt.free(val);
  return FA_OK;
}

void record_stats(fa_ctx* ctx, int64_t cells, int64_t blocks, int64_t nodes, int64_t tile_nodes) {
  float t01 = 0, t12 = 0, t23 = 0;
  cudaEventElapsedTime(&t01, ctx->ev[0], ctx->ev[1]);
  cudaEventElapsedTime(&t12, ctx->ev[1], ctx->ev[2]);
  cudaEventElapsedTime(&t23, ctx->ev[2], ctx->ev[3]);
  fa_stats& S = ctx->stats;
  const double ex = S.ms_exchange;
  const int64_t bx = S.bytes_exchanged;
  S = fa_stats{};
  S.ms_pass1 = t01;
  S.ms_graph = t12;
  S.ms_pass2 = t23;
  S.ms_total = t01 + t12 + t23;
  S.ms_exchange = ex;
  S.bytes_exchanged = bx;
  S.cells = cells;
  S.blocks = blocks;
  S.graph_nodes = nodes;
  S.tile_nodes = tile_nodes;
  S.peel_rounds = ctx->rt.peel_rounds;
  S.contract_levels = ctx->rt.contract_levels;
  S.jump_rounds = ctx->rt.jump_rounds;
  S.launches = ctx->rt.launches;
  float t45 = 0, t56 = 0;
  if (cudaEventElapsedTime(&t45, ctx->ev[4], ctx->ev[5]) != cudaSuccess) t45 = 0;
  if (cudaEventElapsedTime(&t56, ctx->ev[5], ctx->ev[6]) != cudaSuccess) t56 = 0;
  cudaGetLastError();
  S.ms_d8 = t45;
  S.ms_block = t56;
}

void reset_run(fa_ctx* ctx) {
  fa::Runtime& rt = ctx->rt;
  rt.st = ctx->st;
  rt.walk_cap = ctx->opt_walk_cap;
  rt.device_solver = ctx->opt_graph == FA_GRAPH_DEVICE;  // AUTO: the small-raster path of run_acc only
  rt.err = cudaSuccess;
  rt.peel_rounds = rt.contract_levels = rt.jump_rounds = rt.launches = 0;
  rt.d_status = ctx->d_small + 1;
  ctx->stats.ms_exchange = 0;
  ctx->stats.bytes_exchanged = 0;
}

fa_status check_types(fa_ctx* ctx, const float* dem, const uint8_t* dirs, const void* w, fa_wtype wtype,
                      fa_atype atype) {
  if ((dem == nullptr) == (dirs == nullptr))
    return set_err(ctx, FA_E_ARG, "exactly one of dem or dirs must be given");
  const bool ok_combo = ((wtype == FA_W_NONE || wtype == FA_W_U32) && (atype == FA_A_U32 || atype == FA_A_U64)) ||
                        ((wtype == FA_W_F32 || wtype == FA_W_NONE) && atype == FA_A_F64);
  if (!ok_combo) return set_err(ctx, FA_E_ARG, "unsupported (wtype, atype) combination");
  if (wtype != FA_W_NONE && !w) return set_err(ctx, FA_E_ARG, "weights pointer is NULL");
  return FA_OK;
}

}  // namespace