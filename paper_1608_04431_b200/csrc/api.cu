// api.cu -- the C ABI of libfa (include/fa.h) and the host orchestration of
// the hot path:
//   pass 1 (H1-H4 per block) -> graph solve (H5) -> pass 2 (H6),
// plus the tiled / row-strip pipeline (H4-H7) used by fa_perimeter_records,
// fa_accumulate_strips (several strips on one device) and fa_accumulate_dist
// (one strip per rank, NCCL over NVLink):
//   phase A (per strip): pass 1 with halo rows, tile-cut block-exit graph ->
//     A_T, tile roots -> tile perimeter records (F, A, L)
//   exchange: the records of every strip reach every rank
//   phase B (per strip): the producer's global graph over all tile perimeter
//     slots, solved redundantly -> offsets x_T (a_in, D11) ->
//     injected into the strip's tile-cut graph -> pass 2 (EVICT).
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
cudaError_t launch_retain(const Geom& g, const T* x_slot, const uint8_t* dirs, T* acc, cudaStream_t st);
// RETAIN (default): pass 1 stores the block-local accumulation in the output
// and the finalize only walks the entry paths; FA_EVICT=1 selects EVICT
// (pass 2 recomputes the block accumulation with w + x).  P:L79-81, L279-284.
inline bool use_retain() {
  const char* e = getenv("FA_EVICT");
  return !(e && e[0] == '1');
}
cudaError_t launch_d8(const float* dem, const float* dem_up, const float* dem_dn, int64_t H, int64_t W,
                      float nodata, uint8_t* dirs,
                      cudaStream_t st);
cudaError_t launch_g1_parent(cudaStream_t st, uint32_t nn, const uint32_t* tgt, const uint8_t* flags,
                             const uint32_t* slot_root, bool cut, uint32_t* parent);
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
cudaError_t fill_depressions(Runtime& rt, const float* z, int64_t H, int64_t W, float nodata, float* out);
template <class T>
cudaError_t launch_scatter_x(cudaStream_t st, uint32_t nn, const uint32_t* tgt, const uint8_t* flags,
                             const T* S, T* x_slot, bool intra_tile);
template <class T>
cudaError_t launch_fold_leaves(cudaStream_t st, int64_t nslots, const T* x_slot, const uint32_t* slot_root, T* S);
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

// absorption entry points run with the default 32-row blocks whatever the
// FA_BR tuning override says (set for the duration of the call)
thread_local bool g_force_br32 = false;
struct ForceBR32 {
  ForceBR32() { g_force_br32 = true; }
  ~ForceBR32() { g_force_br32 = false; }
};

Geom make_geom(int64_t H, int64_t W, int64_t th, int64_t tw) {
  Geom g{};
  g.H = H;
  g.W = W;
  g.TH = (th > 0 && th < H) ? th : H;
  g.TW = (tw > 0 && tw < W) ? tw : W;
  g.TR = (H + g.TH - 1) / g.TH;
  g.TC = (W + g.TW - 1) / g.TW;
  g.br = kBR;
  g.bc = kBC;
  g.nw = kNW;
  // tuning overrides: FA_WARPS = warps (one block each) per CTA, 1..4;
  // FA_BR = block rows, 16 or 32 (blocks are BR x 32, one per warp)
  if (const char* e = getenv("FA_WARPS")) {
    const int v = atoi(e);
    if (v >= 1 && v <= 4) g.nw = v;
  }
  if (const char* e = getenv("FA_BR")) {
    const int v = atoi(e);
    if ((v == 16 || v == 32) && !g_force_br32) g.br = v;
  }
  g.pb = 2 * (g.br + g.bc) - 4;
  g.regular = (g.TH % g.br == 0 && g.TW % g.bc == 0) ? 1 : 0;
  g.nbt_r = (g.TH + g.br - 1) / g.br;
  g.nbt_c = (g.TW + g.bc - 1) / g.bc;
  g.NBR = g.TR * g.nbt_r;
  g.NBC = g.TC * g.nbt_c;
  g.nblocks = g.NBR * g.NBC;
  g.row0 = 0;
  g.GH = H;
  return g;
}

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
    FA_SYM(errorString, "ncclGetErrorString");
#undef FA_SYM
    return getUniqueId && commInitRank && commDestroy && groupStart && groupEnd && send && recv &&
           broadcast && allReduce && errorString;
  }
};
Nccl& nccl() {
  static Nccl n;
  return n;
}

}  // namespace fa

struct fa_ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  int64_t tile_r = 0, tile_c = 0;
  std::string err;
  fa::Runtime rt;
  fa_stats stats{};
  cudaEvent_t ev[8]{};
  uint32_t* d_small = nullptr;  // [0]=node_count [1]=status [2..3]=wsum(u64) [4..15] scratch
  uint32_t* h_small = nullptr;
  // out-of-core streaming (fa_accumulate_streamed): copy stream + buffer events
  cudaStream_t cs = nullptr, cs_out = nullptr;  // uploads / downloads (PCIe is full duplex)
  cudaEvent_t ev_in[2]{}, ev_used[2]{}, ev_out[2]{};
  // multi-GPU
  ncclComm_t comm = nullptr;
  int rank = -1, nranks = 0;
  unsigned char comm_id[128]{};
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
  a.retain = s.acc != nullptr && fa::use_retain();
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
template <class T, int WK>
fa_status strip_pass1(fa_ctx* ctx, Strip<T>& s, bool cut) {
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
  // its ring.  FA_FUSED=1 (or 1-row halos) keeps D8 fused into pass 1.
  const char* fused_env = getenv("FA_FUSED");
  const bool split = s.dem && !(fused_env && fused_env[0] == '1') && (s.halo2 || (!s.dem_up && !s.dem_dn));
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
__global__ void k_tile_bases(fa::Geom g, int64_t* base) {
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

// phase A tail: A_T at block exits, tile roots, tile perimeter records
template <class T>
fa_status strip_records(fa_ctx* ctx, Strip<T>& s, uint32_t* links, uint8_t* fdir, T* tile_acc,
                        T* tile_f = nullptr) {
  using namespace fa;
  cudaStream_t st = ctx->st;
  Runtime& rt = ctx->rt;
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
      CK(forest_solve_weighted(rt, s.nn, s.parent, s.wv, s.S));
      CK(forest_roots_weighted(rt, s.nn, s.parent, s.wv, s.troot, s.ptroot));
      CK(launch_tile_records<T>(st, s.g, s.nslots, s.dtbase, s.dirs_in(), s.slot_root, s.troot, s.node_flags,
                                s.node_slot, s.S, links + s.slot0, fdir + s.slot0, tile_acc + s.slot0, s.slot_f,
                                s.ptroot, s.alpha, tile_f + s.slot0));
      ++rt.launches;
      return FA_OK;
    }
  }
  CK(launch_fold_leaves<T>(st, s.g.nblocks * s.g.pb, s.x_slot, s.slot_root, s.S));  // leaves raked in pass 1
  ++rt.launches;
  CK(forest_solve<T>(rt, s.nn, s.parent, s.S));  // A_T at every block exit (Alg. 1 on each tile)
  CK(forest_roots(rt, s.nn, s.parent, s.troot));
  CK(launch_tile_records<T>(st, s.g, s.nslots, s.dtbase, s.dirs_in(), s.slot_root, s.troot, s.node_flags,
                            s.node_slot, s.S, links + s.slot0, fdir + s.slot0, tile_acc + s.slot0));
  ++rt.launches;
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
template <class T, int WK>
fa_status strip_finish(fa_ctx* ctx, Strip<T>& s, const T* xT_global) {
  using namespace fa;
  cudaStream_t st = ctx->st;
  Runtime& rt = ctx->rt;
  CK(cudaMemcpyAsync(s.S, s.node_val, s.nn * sizeof(T), cudaMemcpyDeviceToDevice, st));
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
  // leaves first (x_slot holds only their pass-1 values here), then x_T
  CK(launch_fold_leaves<T>(st, s.g.nblocks * s.g.pb, s.x_slot, s.slot_root, s.S));
  ++rt.launches;
  CK(launch_inject_slots<T>(st, s.g, s.nslots, s.dtbase, xT_global + s.slot0, s.slot_root, s.S, s.x_slot));
  ++rt.launches;
  CK(forest_solve<T>(rt, s.nn, s.parent, s.S));  // true A at every block exit
  CK(launch_scatter_x<T>(st, s.nn, s.node_tgt, s.node_flags, s.S, s.x_slot, true));
  ++rt.launches;
  if (s.acc) {
    if (use_retain()) CK(launch_retain<T>(s.g, s.x_slot, s.dirs_in(), s.acc, st));
    else CK(launch_pass2<T, WK>(pass_args<T, WK>(ctx, s), st));
    ++rt.launches;
  }
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
  rt.err = cudaSuccess;
  rt.peel_rounds = rt.contract_levels = rt.jump_rounds = rt.launches = 0;
  rt.d_status = ctx->d_small + 1;
  ctx->stats.ms_exchange = 0;
  ctx->stats.bytes_exchanged = 0;
}

// ---------------------------------------------------------------- single device
struct Records {
  uint32_t* links = nullptr;  // device outputs (fa_perimeter_records)
  void* tile_acc = nullptr;
  void* offsets = nullptr;
  bool want = false;
};

template <class T, int WK>
fa_status run_acc(fa_ctx* ctx, int64_t H, int64_t W, const float* dem, float nodata, const uint8_t* dirs,
                  const void* w, T* acc, Records& rec, int nstrips, const float* alpha = nullptr) {
  using namespace fa;
  cudaStream_t st = ctx->st;
  Runtime& rt = ctx->rt;
  reset_run(ctx);
  CK(cudaMemsetAsync(ctx->d_small, 0, 16 * sizeof(uint32_t), st));
  CK(cudaEventRecord(ctx->ev[0], st));
  const Geom gg = make_geom(H, W, ctx->tile_r, ctx->tile_c);
  if (!rec.want && nstrips <= 1) {
    // On one device every tile is resident, so the per-tile problems and the
    // global perimeter graph are solved jointly as one uncut block-exit graph
    // (identical results: accumulation is linear).  The explicit
    // tile level runs for the records and the strip / multi-GPU paths.
    Strip<T> s;
    s.g = gg;
    s.dem = dem;
    s.dirs = dirs;
    s.w = w;
    s.acc = acc;
    s.nodata = nodata;
    fa_status r = strip_pass1<T, WK>(ctx, s, false);
    if (r != FA_OK) { s.release(rt); return r; }
    CK(cudaEventRecord(ctx->ev[1], st));
    const uint32_t stat = rt.h_cnt[1];
    unsigned long long wsum = 0;
    memcpy(&wsum, &rt.h_cnt[2], 8);
    r = check_status(ctx, stat & ~ST_CYCLE, wsum, std::is_same<T, uint32_t>::value);
    if (r != FA_OK) { s.release(rt); cudaStreamSynchronize(st); return r; }
    CK(cudaMemcpyAsync(s.S, s.node_val, s.nn * sizeof(T), cudaMemcpyDeviceToDevice, st));
    // leaves were raked in pass 1: their values sit in the entry offsets
    CK(launch_fold_leaves<T>(st, s.g.nblocks * s.g.pb, s.x_slot, s.slot_root, s.S));
    ++rt.launches;
    CK(forest_solve<T>(rt, s.nn, s.parent, s.S));
    CK(launch_scatter_x<T>(st, s.nn, s.node_tgt, s.node_flags, s.S, s.x_slot, false));
    ++rt.launches;
    if (rt.err) { s.release(rt); return set_err(ctx, FA_E_CUDA, cudaGetErrorString(rt.err)); }
    CK(cudaEventRecord(ctx->ev[2], st));
    if (use_retain()) CK(launch_retain<T>(s.g, s.x_slot, s.dirs_in(), s.acc, st));
    else CK(launch_pass2<T, WK>(pass_args<T, WK>(ctx, s), st));
    ++rt.launches;
    CK(cudaEventRecord(ctx->ev[3], st));
    s.release(rt);
    CK(rt.read(ctx->d_small + 1, 1));
    r = check_status(ctx, rt.h_cnt[0], 0, false);
    if (r != FA_OK) return r;
    record_stats(ctx, H * W, gg.nblocks, s.nn, 0);
    return FA_OK;
  }
  // ---- tiled / strip pipeline on one device (strips = whole tile rows)
  std::vector<int64_t> hbase;
  const int64_t nslots = tile_perim_total(gg, &hbase);
  uint32_t* links = rt.alloc<uint32_t>(nslots);
  uint8_t* fdir = rt.alloc<uint8_t>(nslots);
  T* tile_acc = rt.alloc<T>(nslots);
  T* xT = rt.alloc<T>(nslots);
  T* tile_f = alpha ? rt.alloc<T>(nslots) : nullptr;  // absorption: path factors per tile slot
  if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
  const int G = nstrips < 1 ? 1 : (int)(nstrips > gg.TR ? gg.TR : nstrips);
  std::vector<Strip<T>> strips(G);
  int64_t blocks = 0, nodes = 0;
  auto cleanup = [&]() {
    for (auto& s : strips) s.release(rt);
    for (void* p : {(void*)links, (void*)fdir, (void*)tile_acc, (void*)xT, (void*)tile_f}) rt.free(p);
  };
  for (int i = 0; i < G; ++i) {
    // strip i: tile rows [i*TR/G, (i+1)*TR/G)
    const int64_t tr0 = gg.TR * i / G, tr1 = gg.TR * (i + 1) / G;
    const int64_t r0 = tr0 * gg.TH, r1 = tr1 * gg.TH < H ? tr1 * gg.TH : H;
    Strip<T>& s = strips[i];
    // same tiles as the whole raster: the strip is whole tile rows (a strip
    // shorter than a tile row is the ragged last tile row itself)
    s.g = make_geom(r1 - r0, W, gg.TH, gg.TW);
    s.row_begin = r0;
    s.nodata = nodata;
    s.dem = dem ? dem + r0 * W : nullptr;
    s.dem_up = dem && r0 > 0 ? dem + (r0 - 1) * W : nullptr;
    s.dem_dn = dem && r1 < H ? dem + r1 * W : nullptr;
    s.dem_up2 = dem && r0 > 1 ? dem + (r0 - 2) * W : nullptr;
    s.dem_dn2 = dem && r1 + 1 < H ? dem + (r1 + 1) * W : nullptr;
    s.halo2 = true;
    s.dirs = dirs ? dirs + r0 * W : nullptr;
    s.dirs_up = dirs && r0 > 0 ? dirs + (r0 - 1) * W : nullptr;
    s.dirs_dn = dirs && r1 < H ? dirs + r1 * W : nullptr;
    s.w = w ? static_cast<const char*>(w) + r0 * W * (WK == 0 ? 0 : 4) : nullptr;
    s.acc = acc ? acc + r0 * W : nullptr;
    s.slot0 = hbase[tr0 * gg.TC];
    s.alpha = alpha ? alpha + r0 * W : nullptr;
    fa_status r = strip_pass1<T, WK>(ctx, s, true);
    if (r != FA_OK) { cleanup(); return r; }
    r = strip_records<T>(ctx, s, links, fdir, tile_acc, tile_f);
    if (r != FA_OK) { cleanup(); return r; }
    blocks += s.g.nblocks;
    nodes += s.nn;
  }
  CK(cudaEventRecord(ctx->ev[1], st));
  CK(rt.read(ctx->d_small + 1, 3));
  {
    unsigned long long wsum = 0;
    memcpy(&wsum, &rt.h_cnt[1], 8);
    fa_status r = check_status(ctx, rt.h_cnt[0] & ~ST_CYCLE, wsum, std::is_same<T, uint32_t>::value);
    if (r != FA_OK) { cleanup(); cudaStreamSynchronize(st); return r; }
  }
  fa_status r = solve_g2<T>(ctx, gg, nslots, hbase, links, fdir, tile_acc, xT, tile_f);
  if (r != FA_OK) { cleanup(); return r; }
  CK(cudaEventRecord(ctx->ev[2], st));
  for (auto& s : strips) {
    r = strip_finish<T, WK>(ctx, s, xT);
    if (r != FA_OK) { cleanup(); return r; }
  }
  CK(cudaEventRecord(ctx->ev[3], st));
  if (rec.want) {
    if (rec.links) CK(cudaMemcpyAsync(rec.links, links, nslots * 4, cudaMemcpyDeviceToDevice, st));
    if (rec.tile_acc) CK(cudaMemcpyAsync(rec.tile_acc, tile_acc, nslots * sizeof(T), cudaMemcpyDeviceToDevice, st));
    if (rec.offsets) CK(cudaMemcpyAsync(rec.offsets, xT, nslots * sizeof(T), cudaMemcpyDeviceToDevice, st));
  }
  cleanup();
  if (rt.err) return set_err(ctx, FA_E_CUDA, cudaGetErrorString(rt.err));
  CK(rt.read(ctx->d_small + 1, 1));
  r = check_status(ctx, rt.h_cnt[0], 0, false);
  if (r != FA_OK) return r;
  record_stats(ctx, H * W, blocks, nodes, nslots);
  return FA_OK;
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

fa_status accumulate_impl(fa_ctx* ctx, int64_t rows, int64_t cols, const float* dem, float nodata,
                          const uint8_t* dirs, const void* w, fa_wtype wtype, void* acc, fa_atype atype,
                          Records& rec, int nstrips) {
  if (!ctx) return FA_E_ARG;
  ctx->err.clear();
  if (rows <= 0 || cols <= 0) return set_err(ctx, FA_E_ARG, "rows and cols must be > 0");
  FS(check_types(ctx, dem, dirs, w, wtype, atype));
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->st;
  const size_t n = (size_t)rows * (size_t)cols;
  const size_t asz = atype == FA_A_U32 ? 4 : 8;
  Staged sdem, sdirs, sw, sacc;
  CK(stage_in(st, dem, n * 4, sdem));
  CK(stage_in(st, dirs, n, sdirs));
  CK(stage_in(st, wtype == FA_W_NONE ? nullptr : w, n * 4, sw));
  CK(stage_out_alloc(st, acc, n * asz, sacc));
  Records drec = rec;
  Staged sl, sa, so;
  const int64_t ns = rec.want ? fa_perimeter_slots(ctx, rows, cols) : 0;
  if (rec.want) {
    CK(stage_out_alloc(st, rec.links, ns * 4, sl));
    CK(stage_out_alloc(st, rec.tile_acc, ns * asz, sa));
    CK(stage_out_alloc(st, rec.offsets, ns * asz, so));
    drec.links = (uint32_t*)sl.dev;
    drec.tile_acc = sa.dev;
    drec.offsets = so.dev;
  }
  const float* d_dem = (const float*)sdem.dev;
  const uint8_t* d_dirs = (const uint8_t*)sdirs.dev;
  fa_status s;
  if (atype == FA_A_U32) {
    s = wtype == FA_W_NONE ? run_acc<uint32_t, 0>(ctx, rows, cols, d_dem, nodata, d_dirs, sw.dev, (uint32_t*)sacc.dev, drec, nstrips)
                           : run_acc<uint32_t, 1>(ctx, rows, cols, d_dem, nodata, d_dirs, sw.dev, (uint32_t*)sacc.dev, drec, nstrips);
  } else if (atype == FA_A_U64) {
    using U = unsigned long long;
    s = wtype == FA_W_NONE ? run_acc<U, 0>(ctx, rows, cols, d_dem, nodata, d_dirs, sw.dev, (U*)sacc.dev, drec, nstrips)
                           : run_acc<U, 1>(ctx, rows, cols, d_dem, nodata, d_dirs, sw.dev, (U*)sacc.dev, drec, nstrips);
  } else {
    s = wtype == FA_W_NONE ? run_acc<double, 0>(ctx, rows, cols, d_dem, nodata, d_dirs, sw.dev, (double*)sacc.dev, drec, nstrips)
                           : run_acc<double, 2>(ctx, rows, cols, d_dem, nodata, d_dirs, sw.dev, (double*)sacc.dev, drec, nstrips);
  }
  if (s == FA_OK) {
    if (sacc.owned) CK(cudaMemcpyAsync(acc, sacc.dev, n * asz, cudaMemcpyDeviceToHost, st));
    if (sl.owned) CK(cudaMemcpyAsync(rec.links, sl.dev, ns * 4, cudaMemcpyDeviceToHost, st));
    if (sa.owned) CK(cudaMemcpyAsync(rec.tile_acc, sa.dev, ns * asz, cudaMemcpyDeviceToHost, st));
    if (so.owned) CK(cudaMemcpyAsync(rec.offsets, so.dev, ns * asz, cudaMemcpyDeviceToHost, st));
  }
  for (Staged* p : {&sdem, &sdirs, &sw, &sacc, &sl, &sa, &so})
    if (p->owned) cudaFreeAsync(p->dev, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (s == FA_OK && e != cudaSuccess) return set_err(ctx, FA_E_CUDA, std::string("stream: ") + cudaGetErrorString(e));
  return s;
}

// ---------------------------------------------------------------- absorption (N3)
// Eq. 1 with a per-cell alpha in [0,1] ("most forms of absorption
// represent a simple extension"), on one device with 32x32 blocks:
// pass 1 scales every push by alpha of the pushing cell and records, per
// entry slot, the product f of alpha along its in-block path before the exit;
// the block-exit graph becomes a forest with multiplicative edges
// (alpha(exit) f(target entry)); the finalize scales the carried offset by
// alpha of every cell it leaves.  Linear in w, so the tiling stays exact.
template <int WK>
fa_status run_absorb(fa_ctx* ctx, int64_t H, int64_t W, const float* dem, float nodata, const uint8_t* dirs,
                     const void* w, const float* alpha, double* acc) {
  using namespace fa;
  using T = double;
  cudaStream_t st = ctx->st;
  Runtime& rt = ctx->rt;
  reset_run(ctx);
  CK(cudaMemsetAsync(ctx->d_small, 0, 16 * sizeof(uint32_t), st));
  CK(cudaEventRecord(ctx->ev[0], st));
  Strip<T> s;
  s.g = make_geom(H, W, ctx->tile_r, ctx->tile_c);
  if (s.g.br != 32 || s.g.bc != 32) return set_err(ctx, FA_E_ARG, "absorption runs with 32x32 blocks");
  s.dem = dem;
  s.dirs = dirs;
  s.w = w;
  s.acc = acc;
  s.nodata = nodata;
  s.alpha = alpha;
  fa_status r = strip_pass1<T, WK>(ctx, s, false);
  if (r != FA_OK) { s.release(rt); return r; }
  CK(cudaEventRecord(ctx->ev[1], st));
  r = check_status(ctx, rt.h_cnt[1] & ~ST_CYCLE, 0, false);
  if (r != FA_OK) { s.release(rt); cudaStreamSynchronize(st); return r; }
  const int64_t slots = s.g.nblocks * s.g.pb;
  double* wv = rt.alloc<double>(s.nn ? s.nn : 1);
  if (rt.err) { s.release(rt); return set_err(ctx, FA_E_NOMEM, "device allocation failed"); }
  CK(cudaMemcpyAsync(s.S, s.node_val, s.nn * sizeof(T), cudaMemcpyDeviceToDevice, st));
  CK(launch_absorb_graph(st, s.nn, slots, s.node_alpha, s.node_tgt, s.slot_f, s.x_slot, s.slot_root, wv, s.S));
  rt.launches += 2;
  CK(forest_solve_weighted(rt, s.nn, s.parent, wv, s.S));
  CK(launch_scatter_x_absorb(st, s.nn, s.node_tgt, s.node_alpha, s.S, s.x_slot, s.node_flags, false));
  ++rt.launches;
  CK(cudaEventRecord(ctx->ev[2], st));
  CK(launch_retain_absorb(s.g, s.x_slot, s.dirs_in(), acc, alpha, st));
  ++rt.launches;
  CK(cudaEventRecord(ctx->ev[3], st));
  rt.free(wv);
  s.release(rt);
  if (rt.err) return set_err(ctx, FA_E_CUDA, cudaGetErrorString(rt.err));
  CK(rt.read(ctx->d_small + 1, 1));
  r = check_status(ctx, rt.h_cnt[0], 0, false);
  if (r != FA_OK) return r;
  record_stats(ctx, H * W, s.g.nblocks, s.nn, 0);
  return FA_OK;
}

// ---------------------------------------------------------------- out-of-core (N2)
// The raster lives in host memory and only one strip of whole tile rows (two,
// double-buffered) is resident at a time: the paper's EVICT strategy
// ("only the producer's information and a single tile need be in
// RAM", P:L255 pass 2 recomputes the tile).  Phase A per strip:
// upload z (+2 halo rows each side) or dirs (+1), and w; D8, pass 1 cut at
// tile edges, tile records into the device-resident perimeter arrays; the
// strip's raster state is dropped.  The producer's graph G2 is solved once
// (H5).  Phase B per strip: upload again, recompute pass 1 (A_T in the
// device strip buffer), inject x_T, solve the strip's tile-cut graph, the
// finalize (H6), download A.  Uploads of strip i+1 (one copy stream) and the
// download of strip i-1 (another: PCIe is full duplex) overlap strip i.
template <class T, int WK>
fa_status run_streamed(fa_ctx* ctx, int64_t H, int64_t W, const float* dem_h, float nodata,
                       const uint8_t* dirs_h, const void* w_h, T* acc_h, int64_t strip_rows,
                       const float* alpha_h = nullptr) {
  using namespace fa;
  cudaStream_t st = ctx->st;
  Runtime& rt = ctx->rt;
  reset_run(ctx);
  if (!ctx->cs) {
    CK(cudaStreamCreateWithFlags(&ctx->cs, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&ctx->cs_out, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      CK(cudaEventCreateWithFlags(&ctx->ev_in[b], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_used[b], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_out[b], cudaEventDisableTiming));
    }
  }
  cudaStream_t cs = ctx->cs;
  CK(cudaMemsetAsync(ctx->d_small, 0, 16 * sizeof(uint32_t), st));
  CK(cudaEventRecord(ctx->ev[0], st));
  const Geom gg = make_geom(H, W, ctx->tile_r, ctx->tile_c);
  // strip height in tile rows: requested, else from free device memory
  // (~40 B per resident cell: two z, w and A buffers plus pass-1 state)
  int64_t sr_tiles;
  if (strip_rows > 0) {
    sr_tiles = (strip_rows + gg.TH - 1) / gg.TH;
  } else {
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    const int64_t rows_fit = (int64_t)((double)fr * 0.6 / (40.0 * (double)W));
    sr_tiles = rows_fit / gg.TH;
  }
  if (sr_tiles < 1) sr_tiles = 1;
  if (sr_tiles > gg.TR) sr_tiles = gg.TR;
  const int64_t nst = (gg.TR + sr_tiles - 1) / sr_tiles;
  const int64_t SRr = sr_tiles * gg.TH;  // rows per strip (the last may be shorter)
  std::vector<int64_t> hbase;
  const int64_t nslots = tile_perim_total(gg, &hbase);
  uint32_t* links = rt.alloc<uint32_t>(nslots);
  uint8_t* fdir = rt.alloc<uint8_t>(nslots);
  T* tile_acc = rt.alloc<T>(nslots);
  T* xT = rt.alloc<T>(nslots);
  T* tile_f = alpha_h ? rt.alloc<T>(nslots) : nullptr;  // absorption: path factors per tile slot
  float* alb[2] = {nullptr, nullptr};                     // absorption: alpha strips
  float* zb[2] = {nullptr, nullptr};
  uint8_t* db[2] = {nullptr, nullptr};
  float* wb[2] = {nullptr, nullptr};
  T* ab[2] = {nullptr, nullptr};
  const bool hasw = WK != 0;
  for (int b = 0; b < 2; ++b) {
    if (dem_h) zb[b] = rt.alloc<float>((size_t)((SRr + 4) * W));
    else db[b] = rt.alloc<uint8_t>((size_t)((SRr + 2) * W));
    if (hasw) wb[b] = rt.alloc<float>((size_t)(SRr * W));
    if (alpha_h) alb[b] = rt.alloc<float>((size_t)(SRr * W));
    ab[b] = rt.alloc<T>((size_t)(SRr * W));
  }
  auto cleanup = [&]() {
    cudaStreamSynchronize(cs);
    cudaStreamSynchronize(ctx->cs_out);
    for (void* p : {(void*)links, (void*)fdir, (void*)tile_acc, (void*)xT, (void*)zb[0], (void*)zb[1], (void*)db[0],
                    (void*)db[1], (void*)wb[0], (void*)wb[1], (void*)ab[0], (void*)ab[1], (void*)tile_f,
                    (void*)alb[0], (void*)alb[1]})
      rt.free(p);
  };
  if (rt.err) { cleanup(); return set_err(ctx, FA_E_NOMEM, "device allocation failed (lower strip_rows)"); }
  auto strip_span = [&](int64_t i, int64_t& r0, int64_t& r1) {
    r0 = i * SRr;
    r1 = r0 + SRr < H ? r0 + SRr : H;
  };
  // enqueue the uploads of strip i into buffer b (after its last reader)
  auto upload = [&](int64_t i, int b) -> fa_status {
    int64_t r0, r1;
    strip_span(i, r0, r1);
    CK(cudaStreamWaitEvent(cs, ctx->ev_used[b], 0));
    if (dem_h) {
      // buffer row k holds raster row r0 - 2 + k (rows off the raster are never read)
      const int64_t a = r0 - 2 > 0 ? r0 - 2 : 0, e = r1 + 2 < H ? r1 + 2 : H;
      CK(cudaMemcpyAsync(zb[b] + (a - (r0 - 2)) * W, dem_h + a * W, (size_t)((e - a) * W) * 4,
                         cudaMemcpyHostToDevice, cs));
    } else {
      const int64_t a = r0 - 1 > 0 ? r0 - 1 : 0, e = r1 + 1 < H ? r1 + 1 : H;
      CK(cudaMemcpyAsync(db[b] + (a - (r0 - 1)) * W, dirs_h + a * W, (size_t)((e - a) * W), cudaMemcpyHostToDevice,
                         cs));
    }
    if (hasw)
      CK(cudaMemcpyAsync(wb[b], static_cast<const float*>(w_h) + r0 * W, (size_t)((r1 - r0) * W) * 4,
                         cudaMemcpyHostToDevice, cs));
    if (alpha_h)
      CK(cudaMemcpyAsync(alb[b], alpha_h + r0 * W, (size_t)((r1 - r0) * W) * 4, cudaMemcpyHostToDevice, cs));
    CK(cudaEventRecord(ctx->ev_in[b], cs));
    return FA_OK;
  };
  auto make_strip = [&](int64_t i, int b, Strip<T>& s) {
    int64_t r0, r1;
    strip_span(i, r0, r1);
    const int64_t h = r1 - r0;
    s.g = make_geom(h, W, gg.TH, gg.TW);
    s.row_begin = r0;
    s.nodata = nodata;
    if (dem_h) {
      const float* z = zb[b] + 2 * W;  // raster row r0
      s.dem = z;
      s.dem_up = r0 > 0 ? z - W : nullptr;
      s.dem_up2 = r0 > 1 ? z - 2 * W : nullptr;
      s.dem_dn = r1 < H ? z + h * W : nullptr;
      s.dem_dn2 = r1 + 1 < H ? z + (h + 1) * W : nullptr;
      s.halo2 = true;
    } else {
      const uint8_t* d = db[b] + W;
      s.dirs = d;
      s.dirs_up = r0 > 0 ? d - W : nullptr;
      s.dirs_dn = r1 < H ? d + h * W : nullptr;
    }
    s.w = hasw ? wb[b] : nullptr;
    s.alpha = alpha_h ? alb[b] : nullptr;
    s.acc = ab[b];  // pass 1 accumulates in place (phase A: scratch)
    s.slot0 = hbase[(r0 / gg.TH) * gg.TC];
  };
  int64_t blocks = 0, nodes = 0;
  // ---- phase A
  FS(upload(0, 0));
  for (int64_t i = 0; i < nst; ++i) {
    const int b = (int)(i & 1);
    if (i + 1 < nst) FS(upload(i + 1, b ^ 1));
    CK(cudaStreamWaitEvent(st, ctx->ev_in[b], 0));
    Strip<T> s;
    make_strip(i, b, s);
    fa_status r = strip_pass1<T, WK>(ctx, s, true);
    if (r == FA_OK) r = strip_records<T>(ctx, s, links, fdir, tile_acc, tile_f);
    blocks += s.g.nblocks;
    nodes += s.nn;
    s.release(rt);
    if (r != FA_OK) { cleanup(); return r; }
    CK(cudaEventRecord(ctx->ev_used[b], st));
  }
  CK(cudaEventRecord(ctx->ev[1], st));
  CK(rt.read(ctx->d_small + 1, 3));
  {
    unsigned long long wsum = 0;
    memcpy(&wsum, &rt.h_cnt[1], 8);
    fa_status r = check_status(ctx, rt.h_cnt[0] & ~ST_CYCLE, wsum, std::is_same<T, uint32_t>::value);
    if (r != FA_OK) { cleanup(); cudaStreamSynchronize(st); return r; }
  }
  fa_status r = solve_g2<T>(ctx, gg, nslots, hbase, links, fdir, tile_acc, xT, tile_f);
  if (r != FA_OK) { cleanup(); return r; }
  CK(cudaEventRecord(ctx->ev[2], st));
  // ---- phase B
  FS(upload(0, 0));
  for (int64_t i = 0; i < nst; ++i) {
    const int b = (int)(i & 1);
    if (i + 1 < nst) FS(upload(i + 1, b ^ 1));
    CK(cudaStreamWaitEvent(st, ctx->ev_in[b], 0));
    if (i >= 2) CK(cudaStreamWaitEvent(st, ctx->ev_out[b], 0));  // A of strip i-2 is downloaded
    Strip<T> s;
    make_strip(i, b, s);
    r = strip_pass1<T, WK>(ctx, s, true);
    if (r == FA_OK) {
      s.nslots = tile_perim_total(s.g, nullptr);
      s.dtbase = rt.alloc<int64_t>((size_t)(s.g.TR * s.g.TC + 1));
      if (rt.err) r = set_err(ctx, FA_E_NOMEM, "device allocation failed");
      else {
        k_tile_bases<<<1, 32, 0, st>>>(s.g, s.dtbase);
        ++rt.launches;
        r = strip_finish<T, WK>(ctx, s, xT);
      }
    }
    s.release(rt);
    if (r != FA_OK) { cleanup(); return r; }
    CK(cudaEventRecord(ctx->ev_used[b], st));
    int64_t r0, r1;
    strip_span(i, r0, r1);
    CK(cudaStreamWaitEvent(ctx->cs_out, ctx->ev_used[b], 0));
    CK(cudaMemcpyAsync(acc_h + r0 * W, ab[b], (size_t)((r1 - r0) * W) * sizeof(T), cudaMemcpyDeviceToHost,
                       ctx->cs_out));
    CK(cudaEventRecord(ctx->ev_out[b], ctx->cs_out));
  }
  CK(cudaStreamWaitEvent(st, ctx->ev_out[(nst - 1) & 1], 0));
  if (nst >= 2) CK(cudaStreamWaitEvent(st, ctx->ev_out[nst & 1], 0));
  CK(cudaEventRecord(ctx->ev[3], st));
  cleanup();
  if (rt.err) return set_err(ctx, FA_E_CUDA, cudaGetErrorString(rt.err));
  CK(rt.read(ctx->d_small + 1, 1));
  r = check_status(ctx, rt.h_cnt[0], 0, false);
  if (r != FA_OK) return r;
  record_stats(ctx, H * W, blocks, nodes, nslots);
  ctx->stats.bytes_exchanged =
      (int64_t)(2 * H * W * ((dem_h ? 4 : 1) + (hasw ? 4 : 0) + (alpha_h ? 4 : 0)) + H * W * (int64_t)sizeof(T));
  CK(cudaStreamSynchronize(st));
  return FA_OK;
}

// ---------------------------------------------------------------- multi-GPU (H7)
template <class T>
ncclDataType_t nccl_type() {
  return std::is_same<T, uint32_t>::value ? ncclUint32 : std::is_same<T, double>::value ? ncclFloat64 : ncclUint64;
}

template <class T, int WK>
fa_status run_dist(fa_ctx* ctx, int64_t GH, int64_t W, int64_t row_begin, int64_t H, const float* dem,
                   float nodata, const uint8_t* dirs, const void* w, T* acc,
                   const float* alpha = nullptr) {
  using namespace fa;
  cudaStream_t st = ctx->st;
  Runtime& rt = ctx->rt;
  Nccl& N = nccl();
  const int rank = ctx->rank, nranks = ctx->nranks;
  reset_run(ctx);
  CK(cudaMemsetAsync(ctx->d_small, 0, 16 * sizeof(uint32_t), st));
  CK(cudaEventRecord(ctx->ev[0], st));
  const Geom gg = make_geom(GH, W, ctx->tile_r, ctx->tile_c);
  if (row_begin % gg.TH != 0 || (row_begin + H != GH && H % gg.TH != 0))
    return set_err(ctx, FA_E_ARG, "strips must consist of whole tile rows");
  cudaEvent_t ex0, ex1;
  cudaEventCreate(&ex0);
  cudaEventCreate(&ex1);
  // ---- C1: halo rows, grouped send/recv: two rows of z each way (D8 of the
  // neighbours' edge rows needs their next row too), or one row of codes
  const size_t esz = dem ? 4 : 1;
  const void* src = dem ? (const void*)dem : (const void*)dirs;
  const int64_t nh = (dem && gg.TH >= 2) ? 2 : 1;  // strips are whole tile rows: >= 2 rows when TH >= 2
  void *up = nullptr, *dn = nullptr;
  if (rank > 0) up = rt.alloc<uint8_t>(nh * W * esz);
  if (rank < nranks - 1) dn = rt.alloc<uint8_t>(nh * W * esz);
  if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
  CK(cudaEventRecord(ex0, st));
  NK(N.groupStart());
  const ncclDataType_t rt_row = dem ? ncclFloat32 : ncclUint8;
  if (rank > 0) {  // our first nh rows up, their last nh rows (rows -nh..-1) down to us
    NK(N.send(src, nh * W, rt_row, rank - 1, ctx->comm, st));
    NK(N.recv(up, nh * W, rt_row, rank - 1, ctx->comm, st));
  }
  if (rank < nranks - 1) {
    NK(N.send(static_cast<const char*>(src) + (H - nh) * W * esz, nh * W, rt_row, rank + 1, ctx->comm, st));
    NK(N.recv(dn, nh * W, rt_row, rank + 1, ctx->comm, st));
  }
  NK(N.groupEnd());
  CK(cudaEventRecord(ex1, st));
  // ---- phase A on this strip
  std::vector<int64_t> hbase;
  const int64_t nslots = tile_perim_total(gg, &hbase);
  uint32_t* links = rt.alloc<uint32_t>(nslots);
  uint8_t* fdir = rt.alloc<uint8_t>(nslots);
  T* tile_acc = rt.alloc<T>(nslots);
  T* xT = rt.alloc<T>(nslots);
  T* tile_f = alpha ? rt.alloc<T>(nslots) : nullptr;  // absorption: path factors per tile slot
  if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
  Strip<T> s;
  s.g = make_geom(H, W, gg.TH, gg.TW);
  s.row_begin = row_begin;
  s.nodata = nodata;
  s.dem = dem;
  s.dirs = dirs;
  // halo buffers: up = rows [-nh, -1], dn = rows [H, H + nh)
  s.dem_up = dem && up ? (const float*)up + (nh - 1) * W : nullptr;
  s.dem_dn = dem ? (const float*)dn : nullptr;
  if (nh == 2) {
    s.dem_up2 = up ? (const float*)up : nullptr;
    s.dem_dn2 = dn ? (const float*)dn + W : nullptr;
    s.halo2 = true;
  }
  s.dirs_up = dem ? nullptr : (const uint8_t*)up;
  s.dirs_dn = dem ? nullptr : (const uint8_t*)dn;
  s.w = w;
  s.acc = acc;
  s.slot0 = hbase[(row_begin / gg.TH) * gg.TC];
  s.alpha = alpha;
  auto cleanup = [&]() {
    s.release(rt);
    for (void* p : {(void*)links, (void*)fdir, (void*)tile_acc, (void*)xT, (void*)tile_f, up, dn}) rt.free(p);
  };
  fa_status r = strip_pass1<T, WK>(ctx, s, true);
  if (r == FA_OK) r = strip_records<T>(ctx, s, links, fdir, tile_acc, tile_f);
  if (r != FA_OK) { cleanup(); return r; }
  CK(cudaEventRecord(ctx->ev[1], st));
  // ---- C3 status all-reduce (max) + C2 exchange of the tile records
  // (every rank's slots are a contiguous range: one broadcast per rank)
  NK(N.allReduce(ctx->d_small + 1, ctx->d_small + 1, 1, ncclUint32, ncclMax, ctx->comm, st));
  std::vector<int64_t> s0(nranks + 1), rows_of(nranks);
  {
    // ranks' first rows: gathered through the same all-reduce trick (one value each)
    int64_t* d = rt.alloc<int64_t>(nranks);
    CK(cudaMemsetAsync(d, 0, nranks * sizeof(int64_t), st));
    CK(cudaMemcpyAsync(d + rank, &row_begin, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    NK(N.allReduce(d, d, nranks, ncclInt64, ncclSum, ctx->comm, st));
    CK(cudaMemcpyAsync(rows_of.data(), d, nranks * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    rt.free(d);
  }
  for (int q = 0; q < nranks; ++q) s0[q] = hbase[(rows_of[q] / gg.TH) * gg.TC];
  s0[nranks] = nslots;
  CK(cudaEventRecord(ex0, st));
  NK(N.groupStart());
  for (int q = 0; q < nranks; ++q) {
    const size_t cnt = (size_t)(s0[q + 1] - s0[q]);
    NK(N.broadcast(links + s0[q], links + s0[q], cnt, ncclUint32, q, ctx->comm, st));
    NK(N.broadcast(fdir + s0[q], fdir + s0[q], cnt, ncclUint8, q, ctx->comm, st));
    NK(N.broadcast(tile_acc + s0[q], tile_acc + s0[q], cnt, nccl_type<T>(), q, ctx->comm, st));
    if (tile_f) NK(N.broadcast(tile_f + s0[q], tile_f + s0[q], cnt, nccl_type<T>(), q, ctx->comm, st));
  }
  NK(N.groupEnd());
  CK(cudaEventRecord(ex1, st));
  CK(rt.read(ctx->d_small + 1, 1));
  r = check_status(ctx, rt.h_cnt[0] & ~ST_CYCLE, 0, false);
  if (r != FA_OK) { cleanup(); return r; }
  // ---- phase B: global graph redundantly on every rank, then this strip
  r = solve_g2<T>(ctx, gg, nslots, hbase, links, fdir, tile_acc, xT, tile_f);
  if (r == FA_OK) {
    CK(cudaEventRecord(ctx->ev[2], st));
    r = strip_finish<T, WK>(ctx, s, xT);
  }
  if (r != FA_OK) { cleanup(); return r; }
  NK(N.allReduce(ctx->d_small + 1, ctx->d_small + 1, 1, ncclUint32, ncclMax, ctx->comm, st));
  CK(cudaEventRecord(ctx->ev[3], st));
  cleanup();
  CK(rt.read(ctx->d_small + 1, 1));
  r = check_status(ctx, rt.h_cnt[0], 0, false);
  float exm = 0;
  cudaEventElapsedTime(&exm, ex0, ex1);
  cudaEventDestroy(ex0);
  cudaEventDestroy(ex1);
  ctx->stats.ms_exchange = exm;
  ctx->stats.bytes_exchanged = (int64_t)(nslots * (4 + 1 + sizeof(T) * (tile_f ? 2 : 1)) + 2 * nh * W * esz);
  if (r != FA_OK) return r;
  record_stats(ctx, H * W, s.g.nblocks, s.nn, nslots);
  return FA_OK;
}

}  // namespace

namespace {
fa_status dist_impl(fa_ctx* ctx, const void* nccl_id128, int rank, int nranks, int64_t global_rows,
                    int64_t cols, int64_t row_begin, int64_t local_rows, const float* dem, float nodata,
                    const uint8_t* dirs, const void* w, fa_wtype wtype, void* acc, fa_atype atype,
                    const float* alpha);
}  // namespace

extern "C" {

fa_status fa_create(fa_ctx** out, int device, void* cuda_stream, int64_t tile_rows, int64_t tile_cols) {
  if (!out) return FA_E_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return FA_E_STATE;
  }
  fa_ctx* c = new fa_ctx();
  c->device = device;
  c->st = (cudaStream_t)cuda_stream;
  c->tile_r = tile_rows;
  c->tile_c = tile_cols;
  if (cudaSetDevice(device) != cudaSuccess) { delete c; return FA_E_CUDA; }
  // keep freed stream-ordered memory cached in the pool between calls
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  for (auto& e : c->ev)
    if (cudaEventCreate(&e) != cudaSuccess) { delete c; return FA_E_CUDA; }
  if (cudaMalloc(&c->d_small, 64 * sizeof(uint32_t)) != cudaSuccess ||
      cudaMallocHost(&c->h_small, 64 * sizeof(uint32_t)) != cudaSuccess) {
    delete c;
    return FA_E_NOMEM;
  }
  c->rt.st = c->st;
  c->rt.h_cnt = c->h_small;
  c->rt.d_cnt = c->d_small + 16;
  *out = c;
  return FA_OK;
}

fa_status fa_destroy(fa_ctx* ctx) {
  if (!ctx) return FA_E_ARG;
  cudaSetDevice(ctx->device);
  if (ctx->st) cudaStreamSynchronize(ctx->st);
  else cudaDeviceSynchronize();
  if (ctx->comm) fa::nccl().commDestroy(ctx->comm);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (int b = 0; b < 2; ++b)
    for (cudaEvent_t e : {ctx->ev_in[b], ctx->ev_used[b], ctx->ev_out[b]})
      if (e) cudaEventDestroy(e);
  if (ctx->cs) cudaStreamDestroy(ctx->cs);
  if (ctx->cs_out) cudaStreamDestroy(ctx->cs_out);
  cudaFree(ctx->d_small);
  cudaFreeHost(ctx->h_small);
  delete ctx;
  return FA_OK;
}

const char* fa_last_error(const fa_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

fa_status fa_flowdirs(fa_ctx* ctx, const float* dem, int64_t rows, int64_t cols, float nodata,
                      uint8_t* dirs) {
  if (!ctx) return FA_E_ARG;
  ctx->err.clear();
  if (!dem || !dirs || rows <= 0 || cols <= 0) return set_err(ctx, FA_E_ARG, "bad arguments");
  CK(cudaSetDevice(ctx->device));
  const size_t n = (size_t)rows * (size_t)cols;
  Staged sd, so;
  CK(stage_in(ctx->st, dem, n * 4, sd));
  CK(stage_out_alloc(ctx->st, dirs, n, so));
  CK(cudaEventRecord(ctx->ev[0], ctx->st));
  CK(fa::launch_d8((const float*)sd.dev, nullptr, nullptr, rows, cols, nodata, (uint8_t*)so.dev, ctx->st));
  CK(cudaEventRecord(ctx->ev[1], ctx->st));
  if (so.owned) CK(cudaMemcpyAsync(dirs, so.dev, n, cudaMemcpyDeviceToHost, ctx->st));
  if (sd.owned) cudaFreeAsync(sd.dev, ctx->st);
  if (so.owned) cudaFreeAsync(so.dev, ctx->st);
  CK(cudaStreamSynchronize(ctx->st));
  float ms = 0;
  cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
  ctx->stats = fa_stats{};
  ctx->stats.ms_total = ctx->stats.ms_pass1 = ms;
  ctx->stats.cells = rows * cols;
  ctx->stats.launches = 1;
  return FA_OK;
}

fa_status fa_fill(fa_ctx* ctx, const float* dem, int64_t rows, int64_t cols, float nodata, float* out) {
  if (!ctx) return FA_E_ARG;
  ctx->err.clear();
  if (!dem || !out || rows <= 0 || cols <= 0) return set_err(ctx, FA_E_ARG, "bad arguments");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->st;
  const size_t n = (size_t)rows * (size_t)cols;
  Staged sz, so;
  CK(stage_in(st, dem, n * 4, sz));
  CK(stage_out_alloc(st, out, n * 4, so));
  reset_run(ctx);
  CK(cudaEventRecord(ctx->ev[0], st));
  cudaError_t e = fa::fill_depressions(ctx->rt, (const float*)sz.dev, rows, cols, nodata, (float*)so.dev);
  CK(cudaEventRecord(ctx->ev[1], st));
  if (e == cudaSuccess && so.owned) e = cudaMemcpyAsync(out, so.dev, n * 4, cudaMemcpyDeviceToHost, st);
  for (Staged* p : {&sz, &so})
    if (p->owned) cudaFreeAsync(p->dev, st);
  const cudaError_t e2 = cudaStreamSynchronize(st);
  if (e != cudaSuccess || e2 != cudaSuccess)
    return set_err(ctx, FA_E_CUDA, std::string("fill: ") + cudaGetErrorString(e != cudaSuccess ? e : e2));
  float ms = 0;
  cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
  ctx->stats = fa_stats{};
  ctx->stats.ms_total = ms;
  ctx->stats.cells = rows * cols;
  ctx->stats.launches = ctx->rt.launches;
  return FA_OK;
}

fa_status fa_accumulate(fa_ctx* ctx, int64_t rows, int64_t cols, const float* dem, float nodata,
                        const uint8_t* dirs, const void* w, fa_wtype wtype, void* acc, fa_atype atype) {
  Records rec;
  if (!acc) return set_err(ctx, FA_E_ARG, "acc is NULL");
  return accumulate_impl(ctx, rows, cols, dem, nodata, dirs, w, wtype, acc, atype, rec, 1);
}

fa_status fa_accumulate_strips(fa_ctx* ctx, int nstrips, int64_t rows, int64_t cols, const float* dem,
                               float nodata, const uint8_t* dirs, const void* w, fa_wtype wtype, void* acc,
                               fa_atype atype) {
  Records rec;
  if (!acc) return set_err(ctx, FA_E_ARG, "acc is NULL");
  if (nstrips < 1) return set_err(ctx, FA_E_ARG, "nstrips must be >= 1");
  return accumulate_impl(ctx, rows, cols, dem, nodata, dirs, w, wtype, acc, atype, rec, nstrips);
}

fa_status fa_accumulate_absorb(fa_ctx* ctx, int nstrips, int64_t rows, int64_t cols, const float* dem,
                               float nodata, const uint8_t* dirs, const void* w, fa_wtype wtype,
                               const float* alpha, double* acc) {
  fa::ForceBR32 force_br32;
  if (!ctx) return FA_E_ARG;
  ctx->err.clear();
  if (rows <= 0 || cols <= 0) return set_err(ctx, FA_E_ARG, "rows and cols must be > 0");
  if (!acc || !alpha) return set_err(ctx, FA_E_ARG, "acc and alpha must be given");
  if (wtype == FA_W_U32) return set_err(ctx, FA_E_ARG, "absorption takes f32 weights or none (f64 output)");
  FS(check_types(ctx, dem, dirs, w, wtype, FA_A_F64));
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->st;
  const size_t n = (size_t)rows * (size_t)cols;
  Staged sdem, sdirs, sw, sal, sacc;
  CK(stage_in(st, dem, n * 4, sdem));
  CK(stage_in(st, dirs, n, sdirs));
  CK(stage_in(st, wtype == FA_W_NONE ? nullptr : w, n * 4, sw));
  CK(stage_in(st, alpha, n * 4, sal));
  CK(stage_out_alloc(st, acc, n * 8, sacc));
  const float* d_dem = (const float*)sdem.dev;
  const uint8_t* d_dirs = (const uint8_t*)sdirs.dev;
  const float* d_al = (const float*)sal.dev;
  fa_status s;
  if (nstrips > 1) {
    // the multi-GPU strip pipeline on this device, with weighted tile links
    Records rec;
    s = wtype == FA_W_NONE
            ? run_acc<double, 0>(ctx, rows, cols, d_dem, nodata, d_dirs, nullptr, (double*)sacc.dev, rec, nstrips, d_al)
            : run_acc<double, 2>(ctx, rows, cols, d_dem, nodata, d_dirs, sw.dev, (double*)sacc.dev, rec, nstrips, d_al);
  } else {
    s = wtype == FA_W_NONE
            ? run_absorb<0>(ctx, rows, cols, d_dem, nodata, d_dirs, nullptr, d_al, (double*)sacc.dev)
            : run_absorb<2>(ctx, rows, cols, d_dem, nodata, d_dirs, sw.dev, d_al, (double*)sacc.dev);
  }
  if (s == FA_OK && sacc.owned) CK(cudaMemcpyAsync(acc, sacc.dev, n * 8, cudaMemcpyDeviceToHost, st));
  for (Staged* p : {&sdem, &sdirs, &sw, &sal, &sacc})
    if (p->owned) cudaFreeAsync(p->dev, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (s == FA_OK && e != cudaSuccess) return set_err(ctx, FA_E_CUDA, std::string("stream: ") + cudaGetErrorString(e));
  return s;
}

fa_status fa_accumulate_absorb_streamed(fa_ctx* ctx, int64_t rows, int64_t cols, const float* dem,
                                        float nodata, const uint8_t* dirs, const void* w, fa_wtype wtype,
                                        const float* alpha, double* acc, int64_t strip_rows) {
  fa::ForceBR32 force_br32;
  if (!ctx) return FA_E_ARG;
  ctx->err.clear();
  if (rows <= 0 || cols <= 0) return set_err(ctx, FA_E_ARG, "rows and cols must be > 0");
  if (!acc || !alpha) return set_err(ctx, FA_E_ARG, "acc and alpha must be given");
  if (wtype == FA_W_U32) return set_err(ctx, FA_E_ARG, "absorption takes f32 weights or none (f64 output)");
  FS(check_types(ctx, dem, dirs, w, wtype, FA_A_F64));
  for (const void* p : {(const void*)dem, (const void*)dirs, w, (const void*)alpha, (const void*)acc})
    if (p && is_device_ptr(p)) return set_err(ctx, FA_E_ARG, "fa_accumulate_absorb_streamed takes host buffers");
  CK(cudaSetDevice(ctx->device));
  return wtype == FA_W_NONE ? run_streamed<double, 0>(ctx, rows, cols, dem, nodata, dirs, w, acc, strip_rows, alpha)
                            : run_streamed<double, 2>(ctx, rows, cols, dem, nodata, dirs, w, acc, strip_rows, alpha);
}

fa_status fa_accumulate_streamed(fa_ctx* ctx, int64_t rows, int64_t cols, const float* dem, float nodata,
                                 const uint8_t* dirs, const void* w, fa_wtype wtype, void* acc, fa_atype atype,
                                 int64_t strip_rows) {
  if (!ctx) return FA_E_ARG;
  ctx->err.clear();
  if (rows <= 0 || cols <= 0) return set_err(ctx, FA_E_ARG, "rows and cols must be > 0");
  if (!acc) return set_err(ctx, FA_E_ARG, "acc is NULL");
  FS(check_types(ctx, dem, dirs, w, wtype, atype));
  for (const void* p : {(const void*)dem, (const void*)dirs, w, (const void*)acc})
    if (p && is_device_ptr(p)) return set_err(ctx, FA_E_ARG, "fa_accumulate_streamed takes host buffers");
  CK(cudaSetDevice(ctx->device));
  if (atype == FA_A_U32) {
    return wtype == FA_W_NONE ? run_streamed<uint32_t, 0>(ctx, rows, cols, dem, nodata, dirs, w, (uint32_t*)acc, strip_rows)
                              : run_streamed<uint32_t, 1>(ctx, rows, cols, dem, nodata, dirs, w, (uint32_t*)acc, strip_rows);
  }
  if (atype == FA_A_U64) {
    using U = unsigned long long;
    return wtype == FA_W_NONE ? run_streamed<U, 0>(ctx, rows, cols, dem, nodata, dirs, w, (U*)acc, strip_rows)
                              : run_streamed<U, 1>(ctx, rows, cols, dem, nodata, dirs, w, (U*)acc, strip_rows);
  }
  return wtype == FA_W_NONE ? run_streamed<double, 0>(ctx, rows, cols, dem, nodata, dirs, w, (double*)acc, strip_rows)
                            : run_streamed<double, 2>(ctx, rows, cols, dem, nodata, dirs, w, (double*)acc, strip_rows);
}

int64_t fa_perimeter_slots(const fa_ctx* ctx, int64_t rows, int64_t cols) {
  if (!ctx || rows <= 0 || cols <= 0) return 0;
  Geom g = fa::make_geom(rows, cols, ctx->tile_r, ctx->tile_c);
  return tile_perim_total(g, nullptr);
}

fa_status fa_perimeter_records(fa_ctx* ctx, int64_t rows, int64_t cols, const float* dem, float nodata,
                               const uint8_t* dirs, const void* w, fa_wtype wtype, fa_atype atype,
                               uint32_t* links, void* tile_acc, void* offsets, void* acc) {
  Records rec;
  rec.want = true;
  rec.links = links;
  rec.tile_acc = tile_acc;
  rec.offsets = offsets;
  return accumulate_impl(ctx, rows, cols, dem, nodata, dirs, w, wtype, acc, atype, rec, 1);
}

fa_status fa_get_stats(const fa_ctx* ctx, fa_stats* out) {
  if (!ctx || !out) return FA_E_ARG;
  *out = ctx->stats;
  return FA_OK;
}

fa_status fa_nccl_unique_id(void* out128) {
  if (!out128) return FA_E_ARG;
  if (!fa::nccl().load()) return FA_E_NCCL;
  ncclUniqueId id;
  if (fa::nccl().getUniqueId(&id) != ncclSuccess) return FA_E_NCCL;
  memcpy(out128, &id, sizeof(id));
  return FA_OK;
}

fa_status fa_accumulate_absorb_dist(fa_ctx* ctx, const void* nccl_id128, int rank, int nranks,
                                    int64_t global_rows, int64_t cols, int64_t row_begin, int64_t local_rows,
                                    const float* dem, float nodata, const uint8_t* dirs, const void* w,
                                    fa_wtype wtype, const float* alpha, double* acc) {
  fa::ForceBR32 force_br32;
  if (!ctx) return FA_E_ARG;
  if (!alpha || !is_device_ptr(alpha)) return set_err(ctx, FA_E_ARG, "alpha must be a device buffer");
  if (wtype == FA_W_U32) return set_err(ctx, FA_E_ARG, "absorption takes f32 weights or none (f64 output)");
  return dist_impl(ctx, nccl_id128, rank, nranks, global_rows, cols, row_begin, local_rows, dem, nodata, dirs, w,
                   wtype, acc, FA_A_F64, alpha);
}

fa_status fa_accumulate_dist(fa_ctx* ctx, const void* nccl_id128, int rank, int nranks, int64_t global_rows,
                             int64_t cols, int64_t row_begin, int64_t local_rows, const float* dem, float nodata,
                             const uint8_t* dirs, const void* w, fa_wtype wtype, void* acc, fa_atype atype) {
  return dist_impl(ctx, nccl_id128, rank, nranks, global_rows, cols, row_begin, local_rows, dem, nodata, dirs, w,
                   wtype, acc, atype, nullptr);
}

}  // extern "C"

namespace {
fa_status dist_impl(fa_ctx* ctx, const void* nccl_id128, int rank, int nranks, int64_t global_rows,
                    int64_t cols, int64_t row_begin, int64_t local_rows, const float* dem, float nodata,
                    const uint8_t* dirs, const void* w, fa_wtype wtype, void* acc, fa_atype atype,
                    const float* alpha) {
  if (!ctx) return FA_E_ARG;
  ctx->err.clear();
  if (!nccl_id128 || nranks < 1 || rank < 0 || rank >= nranks || global_rows <= 0 || cols <= 0 ||
      local_rows <= 0 || row_begin < 0 || row_begin + local_rows > global_rows || !acc)
    return set_err(ctx, FA_E_ARG, "bad arguments");
  FS(check_types(ctx, dem, dirs, w, wtype, atype));
  for (const void* p : {(const void*)dem, (const void*)dirs, (const void*)w, (const void*)acc})
    if (p && !is_device_ptr(p)) return set_err(ctx, FA_E_ARG, "fa_accumulate_dist takes device buffers");
  CK(cudaSetDevice(ctx->device));
  fa::Nccl& N = fa::nccl();
  if (!N.load()) return set_err(ctx, FA_E_NCCL, "cannot load libnccl.so.2");
  if (ctx->comm && (ctx->rank != rank || ctx->nranks != nranks || memcmp(ctx->comm_id, nccl_id128, 128))) {
    N.commDestroy(ctx->comm);
    ctx->comm = nullptr;
  }
  if (!ctx->comm) {
    ncclUniqueId id;
    memcpy(&id, nccl_id128, sizeof(id));
    NK(N.commInitRank(&ctx->comm, nranks, id, rank));
    ctx->rank = rank;
    ctx->nranks = nranks;
    memcpy(ctx->comm_id, nccl_id128, 128);
  }
  fa_status s;
  if (atype == FA_A_U32) {
    s = wtype == FA_W_NONE ? run_dist<uint32_t, 0>(ctx, global_rows, cols, row_begin, local_rows, dem, nodata, dirs, w, (uint32_t*)acc)
                           : run_dist<uint32_t, 1>(ctx, global_rows, cols, row_begin, local_rows, dem, nodata, dirs, w, (uint32_t*)acc);
  } else if (atype == FA_A_U64) {
    using U = unsigned long long;
    s = wtype == FA_W_NONE ? run_dist<U, 0>(ctx, global_rows, cols, row_begin, local_rows, dem, nodata, dirs, w, (U*)acc)
                           : run_dist<U, 1>(ctx, global_rows, cols, row_begin, local_rows, dem, nodata, dirs, w, (U*)acc);
  } else {
    s = wtype == FA_W_NONE ? run_dist<double, 0>(ctx, global_rows, cols, row_begin, local_rows, dem, nodata, dirs, w, (double*)acc, alpha)
                           : run_dist<double, 2>(ctx, global_rows, cols, row_begin, local_rows, dem, nodata, dirs, w, (double*)acc, alpha);
  }
  cudaError_t e = cudaStreamSynchronize(ctx->st);
  if (s == FA_OK && e != cudaSuccess) return set_err(ctx, FA_E_CUDA, std::string("stream: ") + cudaGetErrorString(e));
  return s;
}
}  // namespace
