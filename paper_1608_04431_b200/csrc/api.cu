// api.cu -- the C ABI of libfa (include/fa.h) and the host orchestration of
// the hot path: pass 1 (H1-H4 per block) -> graph solve (H5) -> pass 2 (H6).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>

#include "fa.h"
#include "forest.cuh"

namespace fa {

template <class T, int WK>
cudaError_t launch_pass1(const PassArgs<T, WK>& a, bool from_dem, cudaStream_t st);
template <class T, int WK>
cudaError_t launch_pass2(const PassArgs<T, WK>& a, cudaStream_t st);
cudaError_t launch_d8(const float* dem, int64_t H, int64_t W, float nodata, uint8_t* dirs,
                      cudaStream_t st);
cudaError_t launch_g1_parent(cudaStream_t st, uint32_t nn, const uint32_t* tgt, const uint8_t* flags,
                             const uint32_t* slot_root, bool cut, uint32_t* parent);
template <class T>
cudaError_t launch_scatter_x(cudaStream_t st, uint32_t nn, const uint32_t* tgt, const T* S, T* x_slot);
template <class T>
cudaError_t launch_g2(cudaStream_t st, uint32_t nn, const uint32_t* tgt, const uint8_t* flags,
                      const uint32_t* slot_root, const uint32_t* troot, const T* S1, uint32_t* parent2,
                      T* val2);
template <class T>
cudaError_t launch_inject(cudaStream_t st, uint32_t nn, const uint32_t* tgt, const uint8_t* flags,
                          const uint32_t* slot_root, const T* S2, T* val1, T* xT_slot);
template <class T>
cudaError_t launch_tile_records(cudaStream_t st, const Geom& g, int64_t nslots, const int64_t* tbase,
                                const uint8_t* dirs, const uint32_t* slot_root, const uint32_t* troot,
                                const uint8_t* flags, const uint32_t* node_slot, const T* S1,
                                const T* xT_slot, uint32_t* links, T* tile_acc, T* offs);

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
  // tuning override: FA_BLOCK = 32x32 | 32x64 | 64x64 (block.cu instantiates these)
  if (const char* e = getenv("FA_BLOCK")) {
    if (!strcmp(e, "32x32x1")) { g.nw = 1; }
    else if (!strcmp(e, "32x32x4")) { g.nw = 4; }
    else if (!strcmp(e, "32x64")) { g.br = 32; g.bc = 64; }
    else if (!strcmp(e, "64x64")) { g.br = 64; g.bc = 64; g.nw = 4; }
    else if (!strcmp(e, "64x64x1")) { g.br = 64; g.bc = 64; g.nw = 1; }
    else if (!strcmp(e, "64x64x2")) { g.br = 64; g.bc = 64; g.nw = 2; }
  }
  g.pb = 2 * (g.br + g.bc) - 4;
  g.nbt_r = (g.TH + g.br - 1) / g.br;
  g.nbt_c = (g.TW + g.bc - 1) / g.bc;
  g.NBR = g.TR * g.nbt_r;
  g.NBC = g.TC * g.nbt_c;
  g.nblocks = g.NBR * g.NBC;
  g.row0 = 0;
  g.GH = H;
  return g;
}


}  // namespace fa

struct fa_ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  int64_t tile_r = 0, tile_c = 0;
  std::string err;
  fa::Runtime rt;
  fa_stats stats{};
  cudaEvent_t ev[6]{};
  uint32_t* d_small = nullptr;  // [0]=node_count [1]=status [2..3]=wsum(u64) [4..15] scratch
  uint32_t* h_small = nullptr;
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

template <class T>
constexpr fa_atype atype_of() {
  return std::is_same<T, uint32_t>::value ? FA_A_U32
         : std::is_same<T, double>::value ? FA_A_F64 : FA_A_U64;
}

struct Records {
  uint32_t* links = nullptr;  // device
  void* tile_acc = nullptr;
  void* offsets = nullptr;
  bool want = false;
};

int64_t tile_perim_total(const Geom& g, int64_t* base /* TR*TC+1 or null */) {
  int64_t tot = 0;
  for (int64_t t = 0; t < g.TR * g.TC; ++t) {
    int64_t y0, x0, h, w;
    g.tile_box(t, y0, x0, h, w);
    if (base) base[t] = tot;
    tot += fa::perim_count(h, w);
  }
  if (base) base[g.TR * g.TC] = tot;
  return tot;
}

template <class T, int WK>
fa_status run_acc(fa_ctx* ctx, int64_t H, int64_t W, const float* dem, float nodata,
                  const uint8_t* dirs, const void* w, T* acc, Records& rec) {
  using namespace fa;
  cudaStream_t st = ctx->st;
  Runtime& rt = ctx->rt;
  rt.st = st;
  rt.err = cudaSuccess;
  rt.peel_rounds = rt.contract_levels = rt.jump_rounds = rt.launches = 0;
  Geom g = make_geom(H, W, ctx->tile_r, ctx->tile_c);
  const int64_t slots = g.nblocks * g.pb;
  if (slots >= (int64_t)0xFFFFFFF0ll)
    return set_err(ctx, FA_E_ARG, "raster too large for one device (block slots exceed 2^32)");
  CK(cudaEventRecord(ctx->ev[0], st));
  uint8_t* dirs_buf = nullptr;
  if (dem) {
    CK(cudaMallocAsync(&dirs_buf, (size_t)(H * W), st));
  }
  uint32_t* slot_root = rt.alloc<uint32_t>(slots);
  T* node_val = rt.alloc<T>(slots);
  uint32_t* node_slot = rt.alloc<uint32_t>(slots);
  uint32_t* node_tgt = rt.alloc<uint32_t>(slots);
  uint8_t* node_flags = rt.alloc<uint8_t>(slots);
  T* x_slot = rt.alloc<T>(slots);
  if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
  CK(cudaMemsetAsync(ctx->d_small, 0, 16 * sizeof(uint32_t), st));
  CK(cudaMemsetAsync(x_slot, 0, slots * sizeof(T), st));

  PassArgs<T, WK> a{};
  a.g = g;
  a.dem = dem;
  a.nodata = nodata;
  a.dirs_in = dem ? dirs_buf : dirs;
  a.dirs_out = dirs_buf;
  a.w = w;
  a.node_count = ctx->d_small + 0;
  a.status = ctx->d_small + 1;
  a.wsum = reinterpret_cast<unsigned long long*>(ctx->d_small + 2);
  a.node_val = node_val;
  a.node_slot = node_slot;
  a.node_tgt = node_tgt;
  a.node_flags = node_flags;
  a.slot_root = slot_root;
  a.x_slot = x_slot;
  a.acc = acc;
  rt.d_status = ctx->d_small + 1;
  CK(launch_pass1<T, WK>(a, dem != nullptr, st));
  ++rt.launches;
  CK(cudaEventRecord(ctx->ev[1], st));
  CK(rt.read(ctx->d_small, 4));
  const uint32_t nn = rt.h_cnt[0];
  const uint32_t stat = rt.h_cnt[1];
  unsigned long long wsum = 0;
  memcpy(&wsum, &rt.h_cnt[2], 8);
  fa_status bad = FA_OK;
  std::string msg;
  if (stat & ST_BADCODE) { bad = FA_E_DIRCODE; msg = "direction raster holds a byte outside {0..8,255}"; }
  else if (stat & ST_BADWEIGHT) { bad = FA_E_ARG; msg = "f32 weights must be finite and >= 0"; }
  else if (std::is_same<T, uint32_t>::value && wsum >= 0xFFFFFFFFull) {
    bad = FA_E_OVERFLOW; msg = "sum of weights reaches the u32 range (NoData marker); use u64";
  }
  if (bad != FA_OK) {
    for (void* p : {(void*)dirs_buf, (void*)slot_root, (void*)node_val, (void*)node_slot,
                    (void*)node_tgt, (void*)node_flags, (void*)x_slot})
      rt.free(p);
    cudaStreamSynchronize(st);
    return set_err(ctx, bad, msg);
  }
  // ---------------- graph (H5)
  uint32_t* parent = rt.alloc<uint32_t>(nn);
  T* S = rt.alloc<T>(nn);
  if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
  // On one device every tile is resident, so the per-tile problems and the
  // global perimeter graph are solved jointly as one uncut block-exit graph
  // (identical results: accumulation is linear).  The explicit
  // tile level (cut graph, tile roots, G2, injection) runs when the tile
  // records are requested -- and is the unit of the multi-GPU exchange.
  const bool multi = rec.want;
  if (!multi) {
    CK(launch_g1_parent(st, nn, node_tgt, node_flags, slot_root, false, parent));
    ++rt.launches;
    CK(cudaMemcpyAsync(S, node_val, nn * sizeof(T), cudaMemcpyDeviceToDevice, st));
    CK(forest_solve<T>(rt, nn, parent, S));
    CK(launch_scatter_x<T>(st, nn, node_tgt, S, x_slot));
    ++rt.launches;
  } else {
    uint32_t* troot = rt.alloc<uint32_t>(nn);
    uint32_t* parent2 = rt.alloc<uint32_t>(nn);
    T* S1 = rt.alloc<T>(nn);
    T* S2 = rt.alloc<T>(nn);
    T* xT = rec.want ? rt.alloc<T>(slots) : nullptr;
    if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
    if (xT) CK(cudaMemsetAsync(xT, 0, slots * sizeof(T), st));
    // per-tile problem: G1 with tile-leaving edges cut -> A_T at block exits
    CK(launch_g1_parent(st, nn, node_tgt, node_flags, slot_root, true, parent));
    ++rt.launches;
    CK(cudaMemcpyAsync(S1, node_val, nn * sizeof(T), cudaMemcpyDeviceToDevice, st));
    CK(forest_solve<T>(rt, nn, parent, S1));
    CK(forest_roots(rt, nn, parent, troot));
    // global perimeter graph -> S2 = A at tile exits
    CK(launch_g2<T>(st, nn, node_tgt, node_flags, slot_root, troot, S1, parent2, S2));
    ++rt.launches;
    CK(forest_solve<T>(rt, nn, parent2, S2));
    // offsets x_T injected at tile entries -> true A at every block exit
    CK(cudaMemcpyAsync(S, node_val, nn * sizeof(T), cudaMemcpyDeviceToDevice, st));
    CK(launch_inject<T>(st, nn, node_tgt, node_flags, slot_root, S2, S, xT));
    ++rt.launches;
    CK(forest_solve<T>(rt, nn, parent, S));
    CK(launch_scatter_x<T>(st, nn, node_tgt, S, x_slot));
    ++rt.launches;
    if (rec.want) {
      const int64_t nt = g.TR * g.TC;
      int64_t* hb = new int64_t[nt + 1];
      const int64_t ns = tile_perim_total(g, hb);
      int64_t* db = rt.alloc<int64_t>(nt + 1);
      CK(cudaMemcpyAsync(db, hb, (nt + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
      CK(cudaStreamSynchronize(st));
      delete[] hb;
      CK(launch_tile_records<T>(st, g, ns, db, a.dirs_in, slot_root, troot, node_flags, node_slot,
                                S1, xT, rec.links, (T*)rec.tile_acc, (T*)rec.offsets));
      ++rt.launches;
      rt.free(db);
    }
    for (void* p : {(void*)troot, (void*)parent2, (void*)S1, (void*)S2, (void*)xT}) rt.free(p);
  }
  if (rt.err) return set_err(ctx, FA_E_CUDA, std::string("graph solve: ") + cudaGetErrorString(rt.err));
  CK(cudaEventRecord(ctx->ev[2], st));
  // ---------------- pass 2 (H6)
  if (acc) { CK(launch_pass2<T, WK>(a, st)); ++rt.launches; }
  CK(cudaEventRecord(ctx->ev[3], st));
  for (void* p : {(void*)dirs_buf, (void*)slot_root, (void*)node_val, (void*)node_slot,
                  (void*)node_tgt, (void*)node_flags, (void*)x_slot, (void*)parent, (void*)S})
    rt.free(p);
  CK(rt.read(ctx->d_small + 1, 1));
  if (rt.h_cnt[0] & ST_CYCLE)
    return set_err(ctx, FA_E_CYCLE, "direction graph has a cycle (some cells never retire)");
  float t01 = 0, t12 = 0, t23 = 0;
  cudaEventElapsedTime(&t01, ctx->ev[0], ctx->ev[1]);
  cudaEventElapsedTime(&t12, ctx->ev[1], ctx->ev[2]);
  cudaEventElapsedTime(&t23, ctx->ev[2], ctx->ev[3]);
  ctx->stats.ms_pass1 = t01;
  ctx->stats.ms_graph = t12;
  ctx->stats.ms_pass2 = t23;
  ctx->stats.ms_total = t01 + t12 + t23;
  ctx->stats.cells = H * W;
  ctx->stats.blocks = g.nblocks;
  ctx->stats.graph_nodes = nn;
  ctx->stats.peel_rounds = rt.peel_rounds;
  ctx->stats.contract_levels = rt.contract_levels;
  ctx->stats.jump_rounds = rt.jump_rounds;
  ctx->stats.launches = rt.launches;
  return FA_OK;
}

fa_status accumulate_impl(fa_ctx* ctx, int64_t rows, int64_t cols, const float* dem, float nodata,
                          const uint8_t* dirs, const void* w, fa_wtype wtype, void* acc,
                          fa_atype atype, Records& rec) {
  if (!ctx) return FA_E_ARG;
  ctx->err.clear();
  if (rows <= 0 || cols <= 0) return set_err(ctx, FA_E_ARG, "rows and cols must be > 0");
  if ((dem == nullptr) == (dirs == nullptr))
    return set_err(ctx, FA_E_ARG, "exactly one of dem or dirs must be given");
  const bool ok_combo = ((wtype == FA_W_NONE || wtype == FA_W_U32) &&
                         (atype == FA_A_U32 || atype == FA_A_U64)) ||
                        ((wtype == FA_W_F32 || wtype == FA_W_NONE) && atype == FA_A_F64);
  if (!ok_combo) return set_err(ctx, FA_E_ARG, "unsupported (wtype, atype) combination");
  if (wtype != FA_W_NONE && !w) return set_err(ctx, FA_E_ARG, "weights pointer is NULL");
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
    s = wtype == FA_W_NONE ? run_acc<uint32_t, 0>(ctx, rows, cols, d_dem, nodata, d_dirs, sw.dev, (uint32_t*)sacc.dev, drec)
                           : run_acc<uint32_t, 1>(ctx, rows, cols, d_dem, nodata, d_dirs, sw.dev, (uint32_t*)sacc.dev, drec);
  } else if (atype == FA_A_U64) {
    using U = unsigned long long;
    s = wtype == FA_W_NONE ? run_acc<U, 0>(ctx, rows, cols, d_dem, nodata, d_dirs, sw.dev, (U*)sacc.dev, drec)
                           : run_acc<U, 1>(ctx, rows, cols, d_dem, nodata, d_dirs, sw.dev, (U*)sacc.dev, drec);
  } else {
    s = wtype == FA_W_NONE ? run_acc<double, 0>(ctx, rows, cols, d_dem, nodata, d_dirs, sw.dev, (double*)sacc.dev, drec)
                           : run_acc<double, 2>(ctx, rows, cols, d_dem, nodata, d_dirs, sw.dev, (double*)sacc.dev, drec);
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
  if (s == FA_OK && e != cudaSuccess)
    return set_err(ctx, FA_E_CUDA, std::string("stream: ") + cudaGetErrorString(e));
  return s;
}

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
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
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
  CK(fa::launch_d8((const float*)sd.dev, rows, cols, nodata, (uint8_t*)so.dev, ctx->st));
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
  return FA_OK;
}

fa_status fa_accumulate(fa_ctx* ctx, int64_t rows, int64_t cols, const float* dem, float nodata,
                        const uint8_t* dirs, const void* w, fa_wtype wtype, void* acc, fa_atype atype) {
  Records rec;
  if (!acc) return set_err(ctx, FA_E_ARG, "acc is NULL");
  return accumulate_impl(ctx, rows, cols, dem, nodata, dirs, w, wtype, acc, atype, rec);
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
  return accumulate_impl(ctx, rows, cols, dem, nodata, dirs, w, wtype, acc, atype, rec);
}

fa_status fa_get_stats(const fa_ctx* ctx, fa_stats* out) {
  if (!ctx || !out) return FA_E_ARG;
  *out = ctx->stats;
  return FA_OK;
}

}  // extern "C"
