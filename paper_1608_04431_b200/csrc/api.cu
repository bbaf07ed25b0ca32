// api.cu -- the C ABI of libfa (include/fa.h), single-device entry points:
//   fa_accumulate: pass 1 (H1-H4 per block) -> graph solve (H5) -> finalize
//     (H6) on one uncut block-exit graph;
//   fa_accumulate_strips / fa_perimeter_records: the tiled row-strip pipeline
//     of pipeline.cuh on one device (the paper's tile level: records, G2);
//   fa_accumulate_streamed: out of core (N2); fa_accumulate_absorb (N3);
//     fa_fill (N4); options and statistics.
// The multi-GPU entry points (H7) are in dist.cu.
#include "pipeline.cuh"

namespace fa {

Geom make_geom(int64_t H, int64_t W, int64_t th, int64_t tw, int br) {
  Geom g{};
  g.H = H;
  g.W = W;
  g.TH = (th > 0 && th < H) ? th : H;
  g.TW = (tw > 0 && tw < W) ? tw : W;
  g.TR = (H + g.TH - 1) / g.TH;
  g.TC = (W + g.TW - 1) / g.TW;
  g.br = (br == 16 || br == 64) ? br : kBR;  // blocks are br x 32, one per warp (FA_OPT_BLOCK_ROWS)
  g.bc = kBC;
  g.nw = kNW;
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

}  // namespace fa

namespace {

// ---------------------------------------------------------------- single device
struct Records {
  uint32_t* links = nullptr;  // device outputs (fa_perimeter_records)
  void* tile_acc = nullptr;
  void* offsets = nullptr;
  bool want = false;
};

// block slots up to which the single-device call runs without a host round
// trip (the device solver's scratch is sized for every slot)
constexpr int64_t kSyncFreeSlots = int64_t(1) << 24;

template <class T, int WK>
fa_status run_acc(fa_ctx* ctx, int64_t H, int64_t W, const float* dem, float nodata, const uint8_t* dirs,
                  const void* w, T* acc, Records& rec, int nstrips, const float* alpha = nullptr) {
  using namespace fa;
  cudaStream_t st = ctx->st;
  Runtime& rt = ctx->rt;
  reset_run(ctx);
  CK(cudaMemsetAsync(ctx->d_small, 0, 16 * sizeof(uint32_t), st));
  CK(cudaEventRecord(ctx->ev[0], st));
  // absorption (alpha) runs with 32-row blocks whatever FA_OPT_BLOCK_ROWS says
  // the strip pipeline with strip-level records (FA_OPT_DIST_RECORDS, as the
  // multi-GPU path): each of the nstrips strips is one tile
  const bool strip_tiles = !rec.want && nstrips > 1 && ctx->opt_dist_records == FA_DIST_STRIPS;
  const int64_t sth = strip_tiles ? (H + nstrips - 1) / nstrips : ctx->tile_r;
  const Geom gg = make_geom(H, W, sth, strip_tiles ? W : ctx->tile_c, alpha ? kBR : ctx->opt_br);
  const int64_t slots = gg.nblocks * gg.pb;
  if (!rec.want && nstrips <= 1 && !alpha && ctx->opt_graph != FA_GRAPH_HOST && slots <= kSyncFreeSlots &&
      !ctx->no_sync_free) {
    // Small rasters (cfg0-cfg2 sizes): the same uncut pipeline without a host
    // round trip until the final status read -- the node count stays on the
    // device and the cooperative device solver (forest_dev.cu) reads it there.
    // Data-dependent errors are reported after the whole call.
    Strip<T> s;
    s.g = gg;
    s.dem = dem;
    s.dirs = dirs;
    s.w = w;
    s.acc = acc;
    s.nodata = nodata;
    CK(cudaMemsetAsync(ctx->d_small + 32, 0, 4 * sizeof(uint32_t), st));
    fa_status r = strip_pass1<T, WK>(ctx, s, false, true);
    if (r != FA_OK) { s.release(rt); return r; }
    CK(cudaEventRecord(ctx->ev[1], st));
    const uint32_t* d_nn = ctx->d_small;
    CK(launch_copy_n<T>(st, s.nn, d_nn, s.node_val, s.S));
    CK(launch_fold_leaves<T>(st, slots, s.x_slot, s.slot_root, s.S));
    rt.launches += 2;
    cudaError_t e = forest_solve_device_async<T>(rt, s.nn, d_nn, s.parent, s.S, ctx->d_small + 32);
    if (e == cudaErrorNotSupported) {  // no cooperative launch: the host-driven solver
      cudaGetLastError();
      CK(rt.read(d_nn, 1));
      CK(forest_solve<T>(rt, rt.h_cnt[0], s.parent, s.S));
    } else {
      CK(e);
    }
    CK(launch_scatter_x<T>(st, s.nn, s.node_tgt, s.node_flags, s.S, s.x_slot, false, d_nn));
    ++rt.launches;
    CK(cudaEventRecord(ctx->ev[2], st));
    if (ctx->retain()) CK(launch_retain<T>(s.g, s.x_slot, s.dirs_in(), s.acc, st));
    else CK(launch_pass2<T, WK>(pass_args<T, WK>(ctx, s), st));
    ++rt.launches;
    CK(cudaEventRecord(ctx->ev[3], st));
    s.release(rt);
    CK(rt.read(ctx->d_small, 36));
    const uint32_t nn = rt.h_cnt[0], stat = rt.h_cnt[1];
    unsigned long long wsum = 0;
    memcpy(&wsum, &rt.h_cnt[2], 8);
    rt.contract_levels += rt.h_cnt[32];
    rt.jump_rounds += rt.h_cnt[33];
    rt.peel_rounds += rt.h_cnt[34];
    if (stat & ST_RETRY) {  // the solver's scratch did not fit (never observed): once more, host-driven
      ctx->no_sync_free = true;
      r = run_acc<T, WK>(ctx, H, W, dem, nodata, dirs, w, acc, rec, nstrips, alpha);
      ctx->no_sync_free = false;
      return r;
    }
    r = check_status(ctx, stat, wsum, std::is_same<T, uint32_t>::value);
    if (r != FA_OK) return r;
    record_stats(ctx, H * W, gg.nblocks, nn, 0);
    return FA_OK;
  }
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
    if (ctx->retain()) CK(launch_retain<T>(s.g, s.x_slot, s.dirs_in(), s.acc, st));
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
  const bool joint_ok = !alpha && G > 1;
  uint32_t* par_all = nullptr;  // the strips' parents as one forest (joint_parents)
  auto cleanup = [&]() {
    for (auto& s : strips) s.release(rt);
    for (void* p : {(void*)links, (void*)fdir, (void*)tile_acc, (void*)xT, (void*)tile_f, (void*)par_all}) rt.free(p);
  };
  for (int i = 0; i < G; ++i) {
    // strip i: tile rows [i*TR/G, (i+1)*TR/G)
    const int64_t tr0 = gg.TR * i / G, tr1 = gg.TR * (i + 1) / G;
    const int64_t r0 = tr0 * gg.TH, r1 = tr1 * gg.TH < H ? tr1 * gg.TH : H;
    Strip<T>& s = strips[i];
    // same tiles as the whole raster: the strip is whole tile rows (a strip
    // shorter than a tile row is the ragged last tile row itself)
    s.g = make_geom(r1 - r0, W, gg.TH, gg.TW, gg.br);
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
    r = strip_records<T>(ctx, s, links + s.slot0, fdir + s.slot0, tile_acc + s.slot0,
                         tile_f ? tile_f + s.slot0 : nullptr, joint_ok ? REC_PRE : REC_ALL);
    if (r != FA_OK) { cleanup(); return r; }
    blocks += s.g.nblocks;
    nodes += s.nn;
  }
  // several strips on one device: their graphs as ONE forest (tile roots in
  // phase A, the solve in phase B), so the per-solve launches and host reads
  // are paid once, not once per strip
  uint32_t n_all = 0;
  if (joint_ok) {
    par_all = joint_parents<T>(ctx, strips, &n_all);
    if (rt.err) { cleanup(); return set_err(ctx, FA_E_NOMEM, "device allocation failed"); }
    if (par_all) {
      fa_status r = roots_strips<T>(ctx, strips, par_all, n_all);
      if (r != FA_OK) { cleanup(); return r; }
    } else {
      for (auto& s : strips) CK(forest_roots(rt, s.nn, s.parent, s.troot));
    }
    for (auto& s : strips) {
      fa_status r = strip_records<T>(ctx, s, links + s.slot0, fdir + s.slot0, tile_acc + s.slot0, nullptr, REC_POST);
      if (r != FA_OK) { cleanup(); return r; }
    }
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
  if (joint_ok) {
    // the strips' graphs as one forest: inject every strip, one solve, finish
    for (auto& s : strips) {
      r = strip_finish<T, WK>(ctx, s, xT, FIN_PRE);
      if (r != FA_OK) { cleanup(); return r; }
    }
    if (par_all) {
      r = solve_strips<T>(ctx, strips, par_all, n_all);
      if (r != FA_OK) { cleanup(); return r; }
    } else {
      for (auto& s : strips) CK(forest_solve<T>(rt, s.nn, s.parent, s.S));
    }
    for (auto& s : strips) {
      r = strip_finish<T, WK>(ctx, s, xT, FIN_POST);
      if (r != FA_OK) { cleanup(); return r; }
    }
  } else {
    for (auto& s : strips) {
      r = strip_finish<T, WK>(ctx, s, xT);
      if (r != FA_OK) { cleanup(); return r; }
    }
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
  s.g = make_geom(H, W, ctx->tile_r, ctx->tile_c, kBR);  // absorption: 32x32 blocks
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

// the copy streams and buffer events of the host-buffer pipelines (created on first use)
fa_status ensure_copy_streams(fa_ctx* ctx) {
  if (ctx->cs) return FA_OK;
  CK(cudaStreamCreateWithFlags(&ctx->cs, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&ctx->cs_out, cudaStreamNonBlocking));
  for (int b = 0; b < 2; ++b) {
    CK(cudaEventCreateWithFlags(&ctx->ev_in[b], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_used[b], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_out[b], cudaEventDisableTiming));
  }
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
  FS(ensure_copy_streams(ctx));
  cudaStream_t cs = ctx->cs;
  CK(cudaMemsetAsync(ctx->d_small, 0, 16 * sizeof(uint32_t), st));
  CK(cudaEventRecord(ctx->ev[0], st));
  const Geom gg = make_geom(H, W, ctx->tile_r, ctx->tile_c, alpha_h ? kBR : ctx->opt_br);
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
    s.g = make_geom(h, W, gg.TH, gg.TW, gg.br);
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
    if (r == FA_OK)
      r = strip_records<T>(ctx, s, links + s.slot0, fdir + s.slot0, tile_acc + s.slot0,
                           tile_f ? tile_f + s.slot0 : nullptr);
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

// ---------------------------------------------------------------- batches of host rasters
// Independent rasters of one shape in host memory (the serving case: a queue
// of DEMs, each accumulated as by fa_accumulate).  Two device buffer sets:
// raster i+1 uploads on one copy stream and raster i-1 downloads on another
// (PCIe is full duplex) while raster i runs the single-device pipeline on
// device buffers -- the same kernels, the same results as fa_accumulate.
template <class T, int WK>
fa_status run_batch(fa_ctx* ctx, int count, int64_t H, int64_t W, const float* const* dem_h, float nodata,
                    const uint8_t* const* dirs_h, const void* const* w_h, T* const* acc_h) {
  using namespace fa;
  cudaStream_t st = ctx->st;
  Runtime& rt = ctx->rt;
  FS(ensure_copy_streams(ctx));
  cudaStream_t cs = ctx->cs, co = ctx->cs_out;
  const size_t n = (size_t)H * (size_t)W;
  const bool hasw = WK != 0;
  float* zb[2] = {nullptr, nullptr};
  uint8_t* db[2] = {nullptr, nullptr};
  float* wb[2] = {nullptr, nullptr};
  T* ab[2] = {nullptr, nullptr};
  const int nbuf = count > 1 ? 2 : 1;
  rt.err = cudaSuccess;
  for (int b = 0; b < nbuf; ++b) {
    if (dem_h) zb[b] = rt.alloc<float>(n);
    else db[b] = rt.alloc<uint8_t>(n);
    if (hasw) wb[b] = rt.alloc<float>(n);
    ab[b] = rt.alloc<T>(n);
  }
  cudaEvent_t tb = nullptr, te = nullptr;
  auto cleanup = [&]() {
    cudaStreamSynchronize(cs);
    cudaStreamSynchronize(co);
    for (int b = 0; b < 2; ++b)
      for (void* p : {(void*)zb[b], (void*)db[b], (void*)wb[b], (void*)ab[b]}) rt.free(p);
    cudaStreamSynchronize(st);
    if (tb) cudaEventDestroy(tb);
    if (te) cudaEventDestroy(te);
  };
  if (rt.err) { cleanup(); return set_err(ctx, FA_E_NOMEM, "device allocation failed (two raster buffer sets)"); }
  CK(cudaEventCreate(&tb));
  CK(cudaEventCreate(&te));
  // the buffers are allocated on st: the copy streams start after that
  for (int b = 0; b < 2; ++b) CK(cudaEventRecord(ctx->ev_used[b], st));
  CK(cudaStreamWaitEvent(cs, ctx->ev_used[0], 0));
  CK(cudaEventRecord(tb, cs));
  auto upload = [&](int i, int b) -> fa_status {
    CK(cudaStreamWaitEvent(cs, ctx->ev_used[b], 0));  // raster i-2 is done with buffer set b
    if (dem_h) CK(cudaMemcpyAsync(zb[b], dem_h[i], n * 4, cudaMemcpyHostToDevice, cs));
    else CK(cudaMemcpyAsync(db[b], dirs_h[i], n, cudaMemcpyHostToDevice, cs));
    if (hasw) CK(cudaMemcpyAsync(wb[b], w_h[i], n * 4, cudaMemcpyHostToDevice, cs));
    CK(cudaEventRecord(ctx->ev_in[b], cs));
    return FA_OK;
  };
  fa_stats last{};
  int64_t launches = 0, nodes = 0;
  double ms_kernels = 0;
  fa_status r = upload(0, 0);
  for (int i = 0; i < count && r == FA_OK; ++i) {
    const int b = i % nbuf;
    if (i + 1 < count) r = upload(i + 1, (i + 1) % nbuf);
    if (r != FA_OK) break;
    CK(cudaStreamWaitEvent(st, ctx->ev_in[b], 0));
    if (i >= 2) CK(cudaStreamWaitEvent(st, ctx->ev_out[b], 0));  // raster i-2 is downloaded
    Records rec;
    r = run_acc<T, WK>(ctx, H, W, zb[b], nodata, db[b], wb[b], ab[b], rec, 1);
    if (r != FA_OK) {
      ctx->err = "raster " + std::to_string(i) + ": " + ctx->err;
      break;
    }
    last = ctx->stats;
    launches += last.launches;
    nodes += last.graph_nodes;
    ms_kernels += last.ms_total;
    CK(cudaEventRecord(ctx->ev_used[b], st));
    CK(cudaStreamWaitEvent(co, ctx->ev_used[b], 0));
    CK(cudaMemcpyAsync(acc_h[i], ab[b], n * sizeof(T), cudaMemcpyDeviceToHost, co));
    CK(cudaEventRecord(ctx->ev_out[b], co));
  }
  if (r != FA_OK) { cleanup(); return r; }
  CK(cudaEventRecord(te, co));
  CK(cudaEventSynchronize(te));
  float ms = 0;
  cudaEventElapsedTime(&ms, tb, te);
  cleanup();
  if (rt.err) return set_err(ctx, FA_E_CUDA, cudaGetErrorString(rt.err));
  // batch statistics: cells, nodes and launches summed over the rasters,
  // ms_total from the first upload to the last download, the phases of the
  // last raster, PCIe bytes in bytes_exchanged
  ctx->stats = last;
  ctx->stats.cells = (int64_t)count * H * W;
  ctx->stats.graph_nodes = nodes;
  ctx->stats.launches = launches;
  ctx->stats.ms_total = ms;
  ctx->stats.ms_compute = ms_kernels;
  ctx->stats.bytes_exchanged = (int64_t)count * H * W * ((dem_h ? 4 : 1) + (hasw ? 4 : 0) + (int64_t)sizeof(T));
  return FA_OK;
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
  cudaError_t e = fa::fill_depressions(ctx->rt, (const float*)sz.dev, rows, cols, nodata, (float*)so.dev,
                                       ctx->opt_fill_tile);
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

fa_status fa_accumulate_batch(fa_ctx* ctx, int count, int64_t rows, int64_t cols, const float* const* dem,
                              float nodata, const uint8_t* const* dirs, const void* const* w, fa_wtype wtype,
                              void* const* acc, fa_atype atype) {
  if (!ctx) return FA_E_ARG;
  ctx->err.clear();
  if (count < 0) return set_err(ctx, FA_E_ARG, "count must be >= 0");
  if (count == 0) return FA_OK;
  if (rows <= 0 || cols <= 0) return set_err(ctx, FA_E_ARG, "rows and cols must be > 0");
  if (!acc) return set_err(ctx, FA_E_ARG, "acc is NULL");
  if ((dem == nullptr) == (dirs == nullptr)) return set_err(ctx, FA_E_ARG, "exactly one of dem, dirs must be given");
  if ((wtype == FA_W_NONE) != (w == nullptr)) return set_err(ctx, FA_E_ARG, "w must be given iff wtype != NONE");
  for (int i = 0; i < count; ++i) {
    const void* in = dem ? (const void*)dem[i] : (const void*)dirs[i];
    const void* wi = w ? w[i] : nullptr;
    if (!in || !acc[i] || (w && !wi))
      return set_err(ctx, FA_E_ARG, "raster " + std::to_string(i) + ": NULL buffer");
    FS(check_types(ctx, dem ? dem[i] : nullptr, dirs ? dirs[i] : nullptr, wi, wtype, atype));
    for (const void* p : {in, wi, (const void*)acc[i]})
      if (p && is_device_ptr(p)) return set_err(ctx, FA_E_ARG, "fa_accumulate_batch takes host buffers");
  }
  CK(cudaSetDevice(ctx->device));
  if (atype == FA_A_U32) {
    auto a = reinterpret_cast<uint32_t* const*>(acc);
    return wtype == FA_W_NONE ? run_batch<uint32_t, 0>(ctx, count, rows, cols, dem, nodata, dirs, w, a)
                              : run_batch<uint32_t, 1>(ctx, count, rows, cols, dem, nodata, dirs, w, a);
  }
  if (atype == FA_A_U64) {
    using U = unsigned long long;
    auto a = reinterpret_cast<U* const*>(acc);
    return wtype == FA_W_NONE ? run_batch<U, 0>(ctx, count, rows, cols, dem, nodata, dirs, w, a)
                              : run_batch<U, 1>(ctx, count, rows, cols, dem, nodata, dirs, w, a);
  }
  auto a = reinterpret_cast<double* const*>(acc);
  return wtype == FA_W_NONE ? run_batch<double, 0>(ctx, count, rows, cols, dem, nodata, dirs, w, a)
                            : run_batch<double, 2>(ctx, count, rows, cols, dem, nodata, dirs, w, a);
}

int64_t fa_perimeter_slots(const fa_ctx* ctx, int64_t rows, int64_t cols) {
  if (!ctx || rows <= 0 || cols <= 0) return 0;
  Geom g = fa::make_geom(rows, cols, ctx->tile_r, ctx->tile_c, ctx->opt_br);
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

fa_status fa_get_stats(const fa_ctx* ctx, void* out, int64_t out_bytes) {
  if (!ctx || !out || out_bytes <= 0) return FA_E_ARG;
  // a caller built against a shorter (older) fa_stats gets its prefix only
  const size_t n = (size_t)out_bytes < sizeof(fa_stats) ? (size_t)out_bytes : sizeof(fa_stats);
  memcpy(out, &ctx->stats, n);
  return FA_OK;
}

fa_status fa_set_option(fa_ctx* ctx, int option, int64_t value) {
  if (!ctx) return FA_E_ARG;
  ctx->err.clear();
  switch (option) {
    case FA_OPT_RETENTION:
      if (value != FA_RETAIN && value != FA_EVICT) break;
      ctx->opt_evict = value == FA_EVICT;
      return FA_OK;
    case FA_OPT_D8:
      if (value != FA_D8_SPLIT && value != FA_D8_FUSED) break;
      ctx->opt_fused = value == FA_D8_FUSED;
      return FA_OK;
    case FA_OPT_BLOCK_ROWS:
      if (value != 16 && value != 32 && value != 64) break;
      ctx->opt_br = (int)value;
      return FA_OK;
    case FA_OPT_WALK_CAP:
      if (value < 0 || value > (1 << 20)) break;
      ctx->opt_walk_cap = (int)value;
      return FA_OK;
    case FA_OPT_FILL_TILE:
      if (value != 32 && value != 64) break;
      ctx->opt_fill_tile = (int)value;
      return FA_OK;
    case FA_OPT_VALUES:
      if (value != FA_VALUES_L2 && value != FA_VALUES_SMEM) break;
      ctx->opt_values = (int)value;
      return FA_OK;
    case FA_OPT_GRAPH:
      if (value != FA_GRAPH_HOST && value != FA_GRAPH_DEVICE && value != FA_GRAPH_AUTO) break;
      ctx->opt_graph = (int)value;
      return FA_OK;
    case FA_OPT_DIST_RECORDS:
      if (value != FA_DIST_TILES && value != FA_DIST_STRIPS) break;
      ctx->opt_dist_records = (int)value;
      return FA_OK;
    default:
      return set_err(ctx, FA_E_ARG, "unknown option");
  }
  return set_err(ctx, FA_E_ARG, "option value out of range");
}

fa_status fa_get_option(const fa_ctx* ctx, int option, int64_t* value) {
  if (!ctx || !value) return FA_E_ARG;
  switch (option) {
    case FA_OPT_RETENTION: *value = ctx->opt_evict ? FA_EVICT : FA_RETAIN; return FA_OK;
    case FA_OPT_D8: *value = ctx->opt_fused ? FA_D8_FUSED : FA_D8_SPLIT; return FA_OK;
    case FA_OPT_BLOCK_ROWS: *value = ctx->opt_br; return FA_OK;
    case FA_OPT_WALK_CAP: *value = ctx->opt_walk_cap; return FA_OK;
    case FA_OPT_FILL_TILE: *value = ctx->opt_fill_tile; return FA_OK;
    case FA_OPT_VALUES: *value = ctx->opt_values; return FA_OK;
    case FA_OPT_GRAPH: *value = ctx->opt_graph; return FA_OK;
    case FA_OPT_DIST_RECORDS: *value = ctx->opt_dist_records; return FA_OK;
    default: return FA_E_ARG;
  }
}

}  // extern "C"
