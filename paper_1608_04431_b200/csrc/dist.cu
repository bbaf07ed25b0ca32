// dist.cu -- multi-GPU row strips (H7): one rank per GPU, rank r owns a
// contiguous strip of whole tile rows.  The paper's producer/consumer
// exchange ("the producer ... joins adjoining tile edges and corners
// into a global graph"; per-tile payload (4 sqrt n)(19) B)
// becomes, per call:
//   C0  a control-plane gather of every rank's arguments (strip bounds,
//       types, tiling): all ranks agree on the partition or all return the
//       same error before any data moves;
//   C1  halo rows: two rows of z (or one row of codes) to / from each
//       neighbour strip (D8 needs the true neighbours, and the D8 of the
//       neighbours' edge rows needs their next row);
//       phase A on the strip (pass 1, tile-cut graph, tile records);
//   C3  a control-plane gather of the status flags (bitwise OR) and of the
//       integer weight sum (u32 overflow, D10);
//   C2  ONE device all-gather of fixed-size padded record buffers (links,
//       A_T, [alpha path factors], F of every tile perimeter slot of the
//       rank's strip);
//       the producer graph G2 solved redundantly on every rank (no second
//       exchange), then phase B on the strip;
//   C3' a final gather of the status flags (cycles found in phase B).
// The exchange runs behind a Transport with two implementations: NCCL (one
// process per GPU, fa_accumulate_dist) and a loopback that runs the ranks as
// host threads, each with its own context and stream, exchanging by
// stream-ordered device copies and events (fa_accumulate_dist_loopback) --
// the same run_dist code, so the multi-rank path is testable on one GPU.
#include <algorithm>
#include <condition_variable>
#include <mutex>
#include <thread>

#include "pipeline.cuh"

namespace {

using fa::Geom;

// ---------------------------------------------------------------- transport
struct Transport {
  int rank = 0, nranks = 1;
  virtual ~Transport() = default;
  // control plane: `bytes` host bytes from every rank -> all[nranks * bytes]
  // in rank order.  Synchronous (returns with `all` filled).
  virtual fa_status gather_host(fa_ctx* ctx, const void* mine, void* all, size_t bytes) = 0;
  // C1: send n_sup bytes at s_up to rank-1 and receive n_rup bytes from it
  // into r_up; likewise downward (rank+1).  Zero counts skip.  Stream-ordered
  // on ctx->st.
  virtual fa_status halo(fa_ctx* ctx, const void* s_up, size_t n_sup, void* r_up, size_t n_rup, const void* s_dn,
                         size_t n_sdn, void* r_dn, size_t n_rdn) = 0;
  // C2: recv[q * bytes, (q+1) * bytes) = rank q's send; stream-ordered.
  virtual fa_status allgather(fa_ctx* ctx, const void* send, void* recv, size_t bytes) = 0;
  // this rank leaves the protocol early: wake peers blocked in the transport
  virtual void abort() {}
};

#define NK(...)                                                                                      \
  do {                                                                                               \
    ncclResult_t _r = (__VA_ARGS__);                                                                 \
    if (_r != ncclSuccess)                                                                           \
      return set_err(ctx, FA_E_NCCL, std::string(#__VA_ARGS__ " failed: ") + fa::nccl().errorString(_r)); \
  } while (0)

struct NcclTransport final : Transport {
  ncclComm_t comm = nullptr;
  fa_status gather_host(fa_ctx* ctx, const void* mine, void* all, size_t bytes) override {
    fa::Nccl& N = fa::nccl();
    fa::Runtime& rt = ctx->rt;
    uint8_t* d = rt.alloc<uint8_t>(bytes * nranks);
    if (rt.err) return set_err(ctx, FA_E_NOMEM, "device allocation failed");
    CK(cudaMemcpyAsync(d + rank * bytes, mine, bytes, cudaMemcpyHostToDevice, ctx->st));
    NK(N.allGather(d + rank * bytes, d, bytes, ncclUint8, comm, ctx->st));
    CK(cudaMemcpyAsync(all, d, bytes * nranks, cudaMemcpyDeviceToHost, ctx->st));
    rt.free(d);
    CK(cudaStreamSynchronize(ctx->st));
    return FA_OK;
  }
  fa_status halo(fa_ctx* ctx, const void* s_up, size_t n_sup, void* r_up, size_t n_rup, const void* s_dn,
                 size_t n_sdn, void* r_dn, size_t n_rdn) override {
    fa::Nccl& N = fa::nccl();
    NK(N.groupStart());
    if (rank > 0) {
      if (n_sup) NK(N.send(s_up, n_sup, ncclUint8, rank - 1, comm, ctx->st));
      if (n_rup) NK(N.recv(r_up, n_rup, ncclUint8, rank - 1, comm, ctx->st));
    }
    if (rank < nranks - 1) {
      if (n_sdn) NK(N.send(s_dn, n_sdn, ncclUint8, rank + 1, comm, ctx->st));
      if (n_rdn) NK(N.recv(r_dn, n_rdn, ncclUint8, rank + 1, comm, ctx->st));
    }
    NK(N.groupEnd());
    return FA_OK;
  }
  fa_status allgather(fa_ctx* ctx, const void* send, void* recv, size_t bytes) override {
    NK(fa::nccl().allGather(send, recv, bytes, ncclUint8, comm, ctx->st));
    return FA_OK;
  }
};

// Loopback: the ranks are host threads.  A rank publishes its buffers and a
// "ready" event recorded on its stream; after a barrier every rank enqueues
// the device copies it needs from its peers behind their ready events and
// records "done"; after a second barrier it makes its stream wait for the
// done events of the peers that read its buffers, so no buffer is reused or
// freed while a peer still copies from it.  Nothing on the device waits on
// another rank's kernels (copies and events only).
struct LoopHub {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool poisoned = false;
  std::vector<const void*> p0, p1;
  std::vector<size_t> s0, s1;
  std::vector<cudaEvent_t> ready, done;
  std::vector<std::vector<uint8_t>> blob;
  explicit LoopHub(int n_) : n(n_), p0(n_), p1(n_), s0(n_), s1(n_), ready(n_), done(n_), blob(n_) {}
  bool barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (poisoned) return false;
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    cv.wait(lk, [&] { return gen != g || poisoned; });
    return gen != g;  // completed (a later poison does not undo it)
  }
  void poison() {
    std::lock_guard<std::mutex> lk(m);
    poisoned = true;
    cv.notify_all();
  }
};

struct LoopTransport final : Transport {
  LoopHub* hub = nullptr;
  fa_status broken(fa_ctx* ctx) { return set_err(ctx, FA_E_STATE, "loopback transport: a peer rank left early"); }
  fa_status gather_host(fa_ctx* ctx, const void* mine, void* all, size_t bytes) override {
    hub->blob[rank].assign(static_cast<const uint8_t*>(mine), static_cast<const uint8_t*>(mine) + bytes);
    if (!hub->barrier()) return broken(ctx);
    for (int q = 0; q < nranks; ++q) {
      if (hub->blob[q].size() != bytes) return set_err(ctx, FA_E_STATE, "loopback: control message sizes differ");
      memcpy(static_cast<uint8_t*>(all) + q * bytes, hub->blob[q].data(), bytes);
    }
    if (!hub->barrier()) return broken(ctx);
    return FA_OK;
  }
  fa_status halo(fa_ctx* ctx, const void* s_up, size_t n_sup, void* r_up, size_t n_rup, const void* s_dn,
                 size_t n_sdn, void* r_dn, size_t n_rdn) override {
    cudaStream_t st = ctx->st;
    CK(cudaEventRecord(hub->ready[rank], st));
    hub->p0[rank] = s_up;
    hub->s0[rank] = n_sup;
    hub->p1[rank] = s_dn;
    hub->s1[rank] = n_sdn;
    if (!hub->barrier()) return broken(ctx);
    fa_status r = FA_OK;
    if (rank > 0 && n_rup) {  // rank-1 sends its last rows down to us
      if (hub->s1[rank - 1] != n_rup) r = set_err(ctx, FA_E_STATE, "loopback: halo sizes disagree");
      else {
        CK(cudaStreamWaitEvent(st, hub->ready[rank - 1], 0));
        CK(cudaMemcpyAsync(r_up, hub->p1[rank - 1], n_rup, cudaMemcpyDefault, st));
      }
    }
    if (rank < nranks - 1 && n_rdn) {  // rank+1 sends its first rows up to us
      if (hub->s0[rank + 1] != n_rdn) r = set_err(ctx, FA_E_STATE, "loopback: halo sizes disagree");
      else {
        CK(cudaStreamWaitEvent(st, hub->ready[rank + 1], 0));
        CK(cudaMemcpyAsync(r_dn, hub->p0[rank + 1], n_rdn, cudaMemcpyDefault, st));
      }
    }
    CK(cudaEventRecord(hub->done[rank], st));
    if (!hub->barrier()) return broken(ctx);
    if (rank > 0) CK(cudaStreamWaitEvent(st, hub->done[rank - 1], 0));
    if (rank < nranks - 1) CK(cudaStreamWaitEvent(st, hub->done[rank + 1], 0));
    return r;
  }
  fa_status allgather(fa_ctx* ctx, const void* send, void* recv, size_t bytes) override {
    cudaStream_t st = ctx->st;
    CK(cudaEventRecord(hub->ready[rank], st));
    hub->p0[rank] = send;
    hub->s0[rank] = bytes;
    if (!hub->barrier()) return broken(ctx);
    fa_status r = FA_OK;
    for (int q = 0; q < nranks; ++q) {
      uint8_t* dst = static_cast<uint8_t*>(recv) + q * bytes;
      if (hub->s0[q] != bytes) {
        r = set_err(ctx, FA_E_STATE, "loopback: all-gather sizes disagree");
        continue;
      }
      if (q == rank) {
        if (dst != send) CK(cudaMemcpyAsync(dst, send, bytes, cudaMemcpyDefault, st));
        continue;
      }
      CK(cudaStreamWaitEvent(st, hub->ready[q], 0));
      CK(cudaMemcpyAsync(dst, hub->p0[q], bytes, cudaMemcpyDefault, st));
    }
    CK(cudaEventRecord(hub->done[rank], st));
    if (!hub->barrier()) return broken(ctx);
    for (int q = 0; q < nranks; ++q)
      if (q != rank) CK(cudaStreamWaitEvent(st, hub->done[q], 0));
    return r;
  }
  void abort() override { hub->poison(); }
};

// ---------------------------------------------------------------- control messages
// C0: one rank's call, as every rank must see it
struct DistHdr {
  int64_t global_rows, cols, row_begin, local_rows, tile_r, tile_c;
  int32_t wtype, atype, from_dem, alpha, br, ok, records, pad;
};
// C3: after phase A / at the end
struct DistStat {
  uint32_t status;  // ST_* bits of the rank
  uint32_t err;     // fa_status of a rank-local failure (0: none)
  unsigned long long wsum;  // integer weight sum over the rank's data cells
};

// rank-local failure inside the protocol: remembered, reported at the next
// status gather so that every rank leaves at the same point
struct LocalErr {
  fa_status s = FA_OK;
  std::string msg;
  void set(fa_ctx* ctx, fa_status st) {
    if (s == FA_OK && st != FA_OK) {
      s = st;
      msg = ctx->err;
    }
  }
};

// combine the gathered statuses; every rank returns the same code
fa_status agree(fa_ctx* ctx, const std::vector<DistStat>& all, int self, const LocalErr& le, bool is_u32,
                bool strip_cycle) {
  uint32_t st = 0;
  unsigned long long wsum = 0;
  for (size_t q = 0; q < all.size(); ++q) {
    if (all[q].err) {
      if ((int)q == self) return set_err(ctx, le.s, le.msg);
      return set_err(ctx, (fa_status)all[q].err, "rank " + std::to_string(q) + " failed (see its context)");
    }
    st |= all[q].status;  // the flags are bits: OR, not max
    wsum += all[q].wsum;
  }
  if (strip_cycle) st &= ~fa::ST_CYCLE;
  return check_status(ctx, st, wsum, is_u32);
}

// unpack the gathered record blocks into the global slot arrays
template <class T>
__global__ void k_unpack_records(const uint8_t* __restrict__ recv, size_t block_bytes, int64_t maxcnt,
                                 const int64_t* __restrict__ s0, int nranks, int self, bool has_f, uint32_t* links,
                                 T* tile_acc, T* tile_f, uint8_t* fdir) {
  const int q = blockIdx.y;
  if (q == self) return;  // this rank's records are already in place
  const int64_t a = s0[q], cnt = s0[q + 1] - s0[q];
  const uint8_t* blk = recv + (size_t)q * block_bytes;
  const uint32_t* L = reinterpret_cast<const uint32_t*>(blk);
  const T* A = reinterpret_cast<const T*>(blk + maxcnt * 4);
  const T* F = reinterpret_cast<const T*>(blk + maxcnt * (4 + sizeof(T)));
  const uint8_t* D = blk + maxcnt * (4 + sizeof(T) * (has_f ? 2 : 1));
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
    links[a + i] = L[i];
    tile_acc[a + i] = A[i];
    if (has_f) tile_f[a + i] = F[i];
    fdir[a + i] = D[i];
  }
}

// ---------------------------------------------------------------- the rank's work
template <class T>
ncclDataType_t nccl_type() {
  return std::is_same<T, uint32_t>::value ? ncclUint32 : std::is_same<T, double>::value ? ncclFloat64 : ncclUint64;
}

struct DistCall {
  int64_t GH = 0, W = 0, row_begin = 0, H = 0;
  const float* dem = nullptr;
  float nodata = 0;
  const uint8_t* dirs = nullptr;
  const void* w = nullptr;
  void* acc = nullptr;
  const float* alpha = nullptr;
  std::vector<DistHdr> hdr;  // every rank's call (after C0)
  // C1 receive buffers (nh rows each, allocated before C0 so that every rank
  // knows the halo exchange can proceed); freed by run_dist
  uint8_t* up = nullptr;
  uint8_t* dn = nullptr;
};

template <class T, int WK>
fa_status run_dist(fa_ctx* ctx, Transport& tp, const DistCall& c) {
  using namespace fa;
  cudaStream_t st = ctx->st;
  Runtime& rt = ctx->rt;
  const int rank = tp.rank, nranks = tp.nranks;
  const int64_t GH = c.GH, W = c.W, H = c.H;
  const bool is_u32 = std::is_same<T, uint32_t>::value;
  reset_run(ctx);
  CK(cudaMemsetAsync(ctx->d_small, 0, 16 * sizeof(uint32_t), st));
  CK(cudaEventRecord(ctx->ev[0], st));
  // Record granularity (FA_OPT_DIST_RECORDS): the context's tiles, or each
  // strip as ONE tile (strip-level records): the block-exit
  // graph is then cut only at strip edges, the records are the strips'
  // perimeters and the producer graph G2 has N tiles instead of TR x TC.
  // Strip tiles need equal strips (the last may be shorter); otherwise the
  // context's tiling is used.
  int64_t th = ctx->tile_r, tw = ctx->tile_c;
  if (ctx->opt_dist_records == FA_DIST_STRIPS && nranks > 1) {
    bool equal = true;
    for (int q = 0; q + 1 < nranks; ++q) equal = equal && c.hdr[q].local_rows == c.hdr[0].local_rows;
    if (equal && (nranks == 1 || c.hdr[nranks - 1].local_rows <= c.hdr[0].local_rows)) {
      th = c.hdr[0].local_rows;
      tw = W;
    }
  }
  const Geom gg = make_geom(GH, W, th, tw, c.alpha ? kBR : ctx->opt_br);
  // every rank's first slot, from the agreed partition (C0)
  std::vector<int64_t> hbase;
  const int64_t nslots = tile_perim_total(gg, &hbase);
  std::vector<int64_t> s0(nranks + 1);
  for (int q = 0; q < nranks; ++q) s0[q] = hbase[(c.hdr[q].row_begin / gg.TH) * gg.TC];
  s0[nranks] = nslots;
  int64_t maxcnt = 0;
  for (int q = 0; q < nranks; ++q) maxcnt = std::max(maxcnt, s0[q + 1] - s0[q]);
  maxcnt = (maxcnt + 15) / 16 * 16;  // 16-byte aligned segments
  const bool has_f = c.alpha != nullptr;
  const size_t blk = (size_t)maxcnt * (4 + sizeof(T) * (has_f ? 2 : 1) + 1);
  // ---- allocations (a failure is reported at the first status gather)
  LocalErr le;
  // C1 sizes: nh rows each way (two rows of z, one of codes), at most the
  // sender's rows; row -2 / H+1 off the raster are simply not there
  const size_t esz = c.dem ? 4 : 1;
  const int64_t nh = c.dem ? 2 : 1;
  const int64_t rows_up = rank > 0 ? std::min<int64_t>(nh, c.hdr[rank - 1].local_rows) : 0;
  const int64_t rows_dn = rank < nranks - 1 ? std::min<int64_t>(nh, c.hdr[rank + 1].local_rows) : 0;
  const int64_t send_up = rank > 0 ? std::min<int64_t>(nh, H) : 0;
  const int64_t send_dn = rank < nranks - 1 ? std::min<int64_t>(nh, H) : 0;
  uint8_t* up = c.up;
  uint8_t* dn = c.dn;
  uint32_t* links = rt.alloc<uint32_t>(nslots);
  uint8_t* fdir = rt.alloc<uint8_t>(nslots);
  T* tile_acc = rt.alloc<T>(nslots);
  T* xT = rt.alloc<T>(nslots);
  T* tile_f = has_f ? rt.alloc<T>(nslots) : nullptr;
  uint8_t* sendb = rt.alloc<uint8_t>(blk);
  uint8_t* recvb = rt.alloc<uint8_t>(blk * nranks);
  int64_t* d_s0 = rt.alloc<int64_t>(nranks + 1);
  if (rt.err) le.set(ctx, set_err(ctx, FA_E_NOMEM, "device allocation failed"));
  Strip<T> s;
  auto cleanup = [&]() {
    s.release(rt);
    for (void* p : {(void*)links, (void*)fdir, (void*)tile_acc, (void*)xT, (void*)tile_f, (void*)up, (void*)dn,
                    (void*)sendb, (void*)recvb, (void*)d_s0})
      rt.free(p);
  };
  // ---- C1: halo rows (the receive buffers were agreed on in C0)
  const void* src = c.dem ? (const void*)c.dem : (const void*)c.dirs;
  cudaEvent_t ex0 = ctx->ev[8], ex1 = ctx->ev[9];
  fa_status r = tp.halo(ctx, src, send_up * W * esz, up, rows_up * W * esz,
                        static_cast<const char*>(src) + (H - send_dn) * W * esz, send_dn * W * esz, dn,
                        rows_dn * W * esz);
  if (r != FA_OK) { tp.abort(); cleanup(); return r; }
  // ---- phase A on this strip
  if (le.s == FA_OK) {
    s.g = make_geom(H, W, gg.TH, gg.TW, gg.br);
    s.row_begin = c.row_begin;
    s.nodata = c.nodata;
    s.dem = c.dem;
    s.dirs = c.dirs;
    // up = rows [-rows_up, -1], dn = rows [H, H + rows_dn)
    if (c.dem) {
      s.dem_up = rows_up ? (const float*)up + (rows_up - 1) * W : nullptr;
      s.dem_up2 = rows_up == 2 ? (const float*)up : nullptr;
      s.dem_dn = rows_dn ? (const float*)dn : nullptr;
      s.dem_dn2 = rows_dn == 2 ? (const float*)dn + W : nullptr;
      s.halo2 = true;
    } else {
      s.dirs_up = rows_up ? up : nullptr;
      s.dirs_dn = rows_dn ? dn : nullptr;
    }
    s.w = c.w;
    s.acc = static_cast<T*>(c.acc);
    s.slot0 = s0[rank];
    s.alpha = c.alpha;
    // the rank's records go straight into its send block
    uint32_t* Ls = reinterpret_cast<uint32_t*>(sendb);
    T* As = reinterpret_cast<T*>(sendb + maxcnt * 4);
    T* Fs = has_f ? reinterpret_cast<T*>(sendb + maxcnt * (4 + sizeof(T))) : nullptr;
    uint8_t* Ds = sendb + maxcnt * (4 + sizeof(T) * (has_f ? 2 : 1));
    r = strip_pass1<T, WK>(ctx, s, true);
    if (r == FA_OK) r = strip_records<T>(ctx, s, Ls, Ds, As, Fs);
    if (r == FA_OK && rt.err) r = set_err(ctx, FA_E_CUDA, cudaGetErrorString(rt.err));
    le.set(ctx, r);
  }
  CK(cudaEventRecord(ctx->ev[1], st));
  // ---- C3: status flags + weight sum of every rank
  DistStat mine{0, (uint32_t)le.s, 0};
  if (le.s == FA_OK) {
    if (rt.read(ctx->d_small + 1, 3) == cudaSuccess) {
      mine.status = rt.h_cnt[0];
      memcpy(&mine.wsum, &rt.h_cnt[1], 8);
    } else {
      le.set(ctx, set_err(ctx, FA_E_CUDA, cudaGetErrorString(rt.err)));
      mine.err = (uint32_t)le.s;
    }
  }
  std::vector<DistStat> all(nranks);
  r = tp.gather_host(ctx, &mine, all.data(), sizeof(DistStat));
  if (r != FA_OK) { tp.abort(); cleanup(); return r; }
  r = agree(ctx, all, rank, le, is_u32, true);
  if (r != FA_OK) { cleanup(); cudaStreamSynchronize(st); return r; }
  // ---- C2: one all-gather of the padded record blocks, then scatter them
  // into the global slot arrays (this rank's own block is copied in place)
  CK(cudaEventRecord(ex0, st));
  r = tp.allgather(ctx, sendb, recvb, blk);
  if (r != FA_OK) { tp.abort(); cleanup(); return r; }
  {
    const int64_t cnt = s0[rank + 1] - s0[rank];
    CK(cudaMemcpyAsync(links + s0[rank], sendb, cnt * 4, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(tile_acc + s0[rank], sendb + maxcnt * 4, cnt * sizeof(T), cudaMemcpyDeviceToDevice, st));
    if (has_f)
      CK(cudaMemcpyAsync(tile_f + s0[rank], sendb + maxcnt * (4 + sizeof(T)), cnt * sizeof(T),
                         cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(fdir + s0[rank], sendb + maxcnt * (4 + sizeof(T) * (has_f ? 2 : 1)), cnt,
                       cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(d_s0, s0.data(), (nranks + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((maxcnt + 255) / 256, 1024)), (unsigned)nranks);
    k_unpack_records<T><<<grid, 256, 0, st>>>(recvb, blk, maxcnt, d_s0, nranks, rank, has_f, links, tile_acc, tile_f,
                                              fdir);
    CK(cudaGetLastError());
    ++rt.launches;
  }
  CK(cudaEventRecord(ex1, st));
  float exm = 0;
  // ---- phase B: the producer graph redundantly on every rank, then this strip
  r = solve_g2<T>(ctx, gg, nslots, hbase, links, fdir, tile_acc, xT, tile_f);
  if (cudaEventElapsedTime(&exm, ex0, ex1) != cudaSuccess) exm = 0;
  if (r == FA_OK) {
    CK(cudaEventRecord(ctx->ev[2], st));
    r = strip_finish<T, WK>(ctx, s, xT);
  }
  if (r == FA_OK && rt.err) r = set_err(ctx, FA_E_CUDA, cudaGetErrorString(rt.err));
  le.set(ctx, r);
  CK(cudaEventRecord(ctx->ev[3], st));
  // ---- C3': final status (cycles found by the graph solves)
  mine = DistStat{0, (uint32_t)le.s, 0};
  if (le.s == FA_OK) {
    if (rt.read(ctx->d_small + 1, 1) == cudaSuccess) mine.status = rt.h_cnt[0];
    else {
      le.set(ctx, set_err(ctx, FA_E_CUDA, cudaGetErrorString(rt.err)));
      mine.err = (uint32_t)le.s;
    }
  }
  r = tp.gather_host(ctx, &mine, all.data(), sizeof(DistStat));
  const int64_t nblocks = s.g.nblocks, nn = s.nn;
  cleanup();
  if (r != FA_OK) { tp.abort(); return r; }
  r = agree(ctx, all, rank, le, false, false);
  if (r != FA_OK) return r;
  record_stats(ctx, H * W, nblocks, nn, nslots);
  ctx->stats.ms_exchange = exm;
  ctx->stats.bytes_exchanged = (int64_t)(blk * nranks + (rows_up + rows_dn) * W * esz);
  return FA_OK;
}

// ---------------------------------------------------------------- agreement (C0)
// Validate this rank's arguments, gather every rank's, and check that they
// describe one raster cut into contiguous strips of whole tile rows ordered
// by rank.  All ranks return the same verdict.
fa_status agree_call(fa_ctx* ctx, Transport& tp, DistCall& c, fa_wtype wtype, fa_atype atype, bool local_ok) {
  DistHdr h{c.GH, c.W, c.row_begin, c.H, ctx->tile_r, ctx->tile_c, (int32_t)wtype, (int32_t)atype,
            c.dem != nullptr, c.alpha != nullptr, c.alpha ? fa::kBR : ctx->opt_br, local_ok ? 1 : 0,
            ctx->opt_dist_records, 0};
  const std::string own_err = ctx->err;
  c.hdr.assign(tp.nranks, DistHdr{});
  FS(tp.gather_host(ctx, &h, c.hdr.data(), sizeof(DistHdr)));
  for (int q = 0; q < tp.nranks; ++q)
    if (!c.hdr[q].ok) {
      if (q == tp.rank) return set_err(ctx, FA_E_ARG, own_err);
      return set_err(ctx, FA_E_STATE, "rank " + std::to_string(q) + " rejected its arguments");
    }
  const DistHdr& a = c.hdr[0];
  const Geom gg = fa::make_geom(a.global_rows, a.cols, a.tile_r, a.tile_c, a.br);
  int64_t next = 0;
  for (int q = 0; q < tp.nranks; ++q) {
    const DistHdr& b = c.hdr[q];
    if (b.global_rows != a.global_rows || b.cols != a.cols || b.tile_r != a.tile_r || b.tile_c != a.tile_c ||
        b.wtype != a.wtype || b.atype != a.atype || b.from_dem != a.from_dem || b.alpha != a.alpha || b.br != a.br ||
        b.records != a.records)
      return set_err(ctx, FA_E_STATE, "ranks disagree on the global raster, tiling, types or options (rank " +
                                          std::to_string(q) + ")");
    const bool last = q == tp.nranks - 1;
    if (b.row_begin != next || b.local_rows <= 0 || b.row_begin % gg.TH != 0 ||
        (!last && b.local_rows % gg.TH != 0) || (last && b.row_begin + b.local_rows != b.global_rows))
      return set_err(ctx, FA_E_STATE, "strips must be contiguous whole tile rows ordered by rank (rank " +
                                          std::to_string(q) + ")");
    // a DEM strip sends its two edge rows: every strip but the last holds >= 2
    if (b.from_dem && !last && b.local_rows < 2)
      return set_err(ctx, FA_E_ARG, "with a DEM, every strip but the last needs at least 2 rows");
    next = b.row_begin + b.local_rows;
  }
  return FA_OK;
}

fa_status dist_run(fa_ctx* ctx, Transport& tp, int64_t global_rows, int64_t cols, int64_t row_begin,
                   int64_t local_rows, const float* dem, float nodata, const uint8_t* dirs, const void* w,
                   fa_wtype wtype, void* acc, fa_atype atype, const float* alpha) {
  ctx->err.clear();
  // rank-local validation: reported through the agreement, never a lone return
  bool ok = true;
  if (global_rows <= 0 || cols <= 0 || local_rows <= 0 || row_begin < 0 || row_begin + local_rows > global_rows ||
      !acc) {
    set_err(ctx, FA_E_ARG, "bad arguments");
    ok = false;
  }
  if (ok && check_types(ctx, dem, dirs, w, wtype, atype) != FA_OK) ok = false;
  if (ok && alpha && wtype == FA_W_U32) {
    set_err(ctx, FA_E_ARG, "absorption takes f32 weights or none (f64 output)");
    ok = false;
  }
  if (ok)
    for (const void* p : {(const void*)dem, (const void*)dirs, (const void*)w, (const void*)acc, (const void*)alpha})
      if (p && !is_device_ptr(p)) {
        set_err(ctx, FA_E_ARG, "the multi-GPU entry points take device buffers");
        ok = false;
        break;
      }
  if (cudaSetDevice(ctx->device) != cudaSuccess) {
    set_err(ctx, FA_E_CUDA, "cudaSetDevice failed");
    ok = false;
  }
  // C1 receive buffers: at most nh rows from each neighbour
  fa::Runtime& rt = ctx->rt;
  rt.st = ctx->st;
  rt.err = cudaSuccess;
  const int64_t nh = dem ? 2 : 1;
  const size_t hb = ok ? (size_t)(nh * cols * (dem ? 4 : 1)) : 0;
  DistCall c;
  c.up = ok && tp.rank > 0 ? rt.alloc<uint8_t>(hb) : nullptr;
  c.dn = ok && tp.rank < tp.nranks - 1 ? rt.alloc<uint8_t>(hb) : nullptr;
  if (ok && rt.err) {
    set_err(ctx, FA_E_NOMEM, "device allocation failed");
    ok = false;
  }
  c.GH = global_rows;
  c.W = cols;
  c.row_begin = row_begin;
  c.H = local_rows;
  c.dem = dem;
  c.nodata = nodata;
  c.dirs = dirs;
  c.w = w;
  c.acc = acc;
  c.alpha = alpha;
  fa_status s = agree_call(ctx, tp, c, wtype, atype, ok);
  if (s != FA_OK) {
    rt.free(c.up);
    rt.free(c.dn);
    cudaStreamSynchronize(ctx->st);
    return s;
  }
  if (atype == FA_A_U32) {
    s = wtype == FA_W_NONE ? run_dist<uint32_t, 0>(ctx, tp, c) : run_dist<uint32_t, 1>(ctx, tp, c);
  } else if (atype == FA_A_U64) {
    using U = unsigned long long;
    s = wtype == FA_W_NONE ? run_dist<U, 0>(ctx, tp, c) : run_dist<U, 1>(ctx, tp, c);
  } else {
    s = wtype == FA_W_NONE ? run_dist<double, 0>(ctx, tp, c) : run_dist<double, 2>(ctx, tp, c);
  }
  // a rank that left before the last collective (a CUDA API failure) must not
  // leave its peers waiting in the transport
  if (s != FA_OK) tp.abort();
  cudaError_t e = cudaStreamSynchronize(ctx->st);
  if (s == FA_OK && e != cudaSuccess) return set_err(ctx, FA_E_CUDA, std::string("stream: ") + cudaGetErrorString(e));
  return s;
}

fa_status dist_nccl(fa_ctx* ctx, const void* nccl_id128, int rank, int nranks, int64_t global_rows, int64_t cols,
                    int64_t row_begin, int64_t local_rows, const float* dem, float nodata, const uint8_t* dirs,
                    const void* w, fa_wtype wtype, void* acc, fa_atype atype, const float* alpha) {
  if (!ctx) return FA_E_ARG;
  ctx->err.clear();
  if (!nccl_id128 || nranks < 1 || rank < 0 || rank >= nranks)
    return set_err(ctx, FA_E_ARG, "bad rank / nranks / NCCL id");
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
  NcclTransport tp;
  tp.rank = rank;
  tp.nranks = nranks;
  tp.comm = ctx->comm;
  return dist_run(ctx, tp, global_rows, cols, row_begin, local_rows, dem, nodata, dirs, w, wtype, acc, atype, alpha);
}

}  // namespace

extern "C" {

fa_status fa_nccl_unique_id(void* out128) {
  if (!out128) return FA_E_ARG;
  if (!fa::nccl().load()) return FA_E_NCCL;
  ncclUniqueId id;
  if (fa::nccl().getUniqueId(&id) != ncclSuccess) return FA_E_NCCL;
  memcpy(out128, &id, sizeof(id));
  return FA_OK;
}

fa_status fa_accumulate_dist(fa_ctx* ctx, const void* nccl_id128, int rank, int nranks, int64_t global_rows,
                             int64_t cols, int64_t row_begin, int64_t local_rows, const float* dem, float nodata,
                             const uint8_t* dirs, const void* w, fa_wtype wtype, void* acc, fa_atype atype) {
  return dist_nccl(ctx, nccl_id128, rank, nranks, global_rows, cols, row_begin, local_rows, dem, nodata, dirs, w,
                   wtype, acc, atype, nullptr);
}

fa_status fa_accumulate_absorb_dist(fa_ctx* ctx, const void* nccl_id128, int rank, int nranks,
                                    int64_t global_rows, int64_t cols, int64_t row_begin, int64_t local_rows,
                                    const float* dem, float nodata, const uint8_t* dirs, const void* w,
                                    fa_wtype wtype, const float* alpha, double* acc) {
  if (!ctx) return FA_E_ARG;
  if (!alpha) return set_err(ctx, FA_E_ARG, "alpha must be given");
  return dist_nccl(ctx, nccl_id128, rank, nranks, global_rows, cols, row_begin, local_rows, dem, nodata, dirs, w,
                   wtype, acc, FA_A_F64, alpha);
}

fa_status fa_accumulate_dist_loopback(fa_ctx* const* ctxs, int nranks, int64_t global_rows, int64_t cols,
                                      const int64_t* row_begin, const int64_t* local_rows,
                                      const float* const* dem, float nodata, const uint8_t* const* dirs,
                                      const void* const* w, fa_wtype wtype, const float* const* alpha,
                                      void* const* acc, fa_atype atype) {
  if (!ctxs || nranks < 1 || !row_begin || !local_rows || !acc) return FA_E_ARG;
  for (int q = 0; q < nranks; ++q) {
    if (!ctxs[q]) return FA_E_ARG;
    for (int p = 0; p < q; ++p)
      if (ctxs[p] == ctxs[q]) return set_err(ctxs[q], FA_E_ARG, "loopback: one context per rank");
  }
  LoopHub hub(nranks);
  std::vector<LoopTransport> tps(nranks);
  fa_status st = FA_OK;
  for (int q = 0; q < nranks && st == FA_OK; ++q) {
    tps[q].rank = q;
    tps[q].nranks = nranks;
    tps[q].hub = &hub;
    fa_ctx* ctx = ctxs[q];
    if (cudaSetDevice(ctx->device) != cudaSuccess ||
        cudaEventCreateWithFlags(&hub.ready[q], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&hub.done[q], cudaEventDisableTiming) != cudaSuccess)
      st = set_err(ctx, FA_E_CUDA, "loopback: event creation failed");
  }
  std::vector<fa_status> res(nranks, FA_OK);
  if (st == FA_OK) {
    std::vector<std::thread> th;
    th.reserve(nranks);
    for (int q = 0; q < nranks; ++q)
      th.emplace_back([&, q]() {
        fa_ctx* ctx = ctxs[q];
        cudaSetDevice(ctx->device);
        res[q] = dist_run(ctx, tps[q], global_rows, cols, row_begin[q], local_rows[q], dem ? dem[q] : nullptr,
                          nodata, dirs ? dirs[q] : nullptr, w ? w[q] : nullptr, wtype, acc[q], atype,
                          alpha ? alpha[q] : nullptr);
      });
    for (auto& t : th) t.join();
    for (int q = 0; q < nranks; ++q)
      if (res[q] != FA_OK) {
        st = res[q];
        break;
      }
  }
  for (int q = 0; q < nranks; ++q) {
    if (hub.ready[q]) cudaEventDestroy(hub.ready[q]);
    if (hub.done[q]) cudaEventDestroy(hub.done[q]);
  }
  return st;
}

}  // extern "C"
