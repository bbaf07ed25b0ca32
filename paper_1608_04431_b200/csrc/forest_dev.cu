// forest_dev.cu -- the forest solver of forest.cu (walks, wide rounds, chain
// contraction, recursion on the segment forest, expansion) as ONE cooperative
// persistent kernel: every decision that forest.cu takes on the host after a
// device-to-host read (frontier size, residual size, pointer-jumping
// convergence, segment count, recursion depth) is taken here by every thread
// from device counters read after a grid-wide barrier, so a solve is one
// launch with no host round trip.  The paper solves its global graph "using
// the same strategy described in Algorithm 1"; the producer's time
// is "negligible".
//
// All threads execute the same control flow (the counters they read after a
// barrier are equal), so grid.sync() is reached uniformly.  Counters are
// written in one phase and read after the next barrier; a counter is reset
// only after a barrier that follows every read of it.  Scratch comes from a
// pool the host sizes from n; a level that would not fit sets a flag and the
// host reruns the solve with forest.cu (never observed: the residual after
// the walks is a small fraction of the nodes).
//
// Measured (FA_OPT_GRAPH = device vs the host-driven default): cfg3 32768^2
// 3.15 vs 1.54 ms (9.26 M nodes), cfg1 8192^2 0.41 vs 0.41 ms, cfg2 0.49 vs
// 0.51 ms, the 8-strip pipeline 31.7 vs 29.2 ms: one persistent grid keeps
// fewer L2-latency-bound walks in flight than the host-driven launches, and
// the host round trips it removes were not the bottleneck.
#include <cooperative_groups.h>

#include <algorithm>

#include <cuda/atomic>

#include "forest.cuh"

namespace cg = cooperative_groups;

namespace fa {
namespace {

#ifndef FA_FOREST_PER_SM
#define FA_FOREST_PER_SM 0  // cooperative CTAs per SM (0: as many as fit)
#endif
#ifndef FA_FOREST_MINB
#define FA_FOREST_MINB 8  // CTAs of 256 per SM: 2048 resident threads (the walks are latency-bound)
#endif
constexpr int kDevMaxLevels = 32;
constexpr int kDevMaxJump = 40;
constexpr uint64_t kDevContractRatio = 8;
// leaves this few relative to the nodes: a chain-dominated forest (cfg2's
// serpentine), contracted at once instead of walked leaf by leaf
constexpr uint64_t kDevLeafRatio = 64;

template <class T>
struct DevLevel {
  uint32_t m;        // residual nodes of the level
  uint32_t* R;       // residual index -> node
  uint32_t* nxt;     // jump pointer: the segment start of each residual node
  T* acc;            // prefix from the node to its segment start (affine acc with WG)
  T* mul;            // WG: product of edge weights along that prefix
  uint32_t* sid;     // residual index -> segment id
  T* val;            // the level's values (expanded from the next level's)
  T* sval;           // the next level's values (segment sums)
};

template <class T, bool WG>
struct DevArgs {
  uint32_t n0;
  const uint32_t* parent0;
  T* val0;
  const T* wv0;
  uint32_t* cnt;      // n0: pending children
  uint8_t* done;      // n0
  uint8_t* one;       // n0: the node has exactly one child (walk fast path)
  uint32_t* fa;       // n0: frontier lists
  uint32_t* fb;
  uint32_t* rid;      // n0: node -> residual index
  uint32_t* ctr;      // 64 counters
  uint8_t* pool;
  size_t pool_bytes;
  DevLevel<T>* lv;    // [kDevMaxLevels]
  uint32_t* status;   // ST_CYCLE
  int cap;            // walk cap (steps before re-queueing)
  const uint32_t* n_dev;  // optional: the node count in device memory (n0 is then a bound)
  uint32_t* stats_out;    // optional: levels, jump rounds, walk rounds (async solves); overflow -> ST_RETRY
};

// counters
enum : int {
  C_F = 0,         // [0..2] frontier counts (3 rotating slots)
  C_RET = 4,       // [4..5] retired nodes of the level (u64)
  C_M = 8,         // residual nodes
  C_MS = 9,        // segments
  C_CH = 10,       // [10..12] pointer-jumping "changed" flags (3 rotating slots)
  C_OVF = 16,      // pool overflow -> host fallback
  C_STATS = 17,    // [17..19] contraction levels, pointer-jumping rounds, walk rounds (Runtime stats)
};

__device__ __forceinline__ uint32_t ld(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ unsigned long long ld64(const uint32_t* p) {
  return __ldcg(reinterpret_cast<const unsigned long long*>(p));
}

// warp-aggregated append; every thread of the warp calls it
__device__ __forceinline__ void append(bool pred, uint32_t v, uint32_t* list, uint32_t* count) {
  const unsigned mask = __ballot_sync(0xFFFFFFFFu, pred);
  if (!mask) return;
  const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(count, (uint32_t)__popc(mask));
  base = __shfl_sync(0xFFFFFFFFu, base, leader);
  if (pred) list[base + __popc(mask & ((1u << lane) - 1))] = v;
}

template <class T>
__device__ __forceinline__ T* carve(uint8_t* pool, size_t& off, size_t count, size_t cap, bool& ovf) {
  off = (off + 15) & ~(size_t)15;
  T* p = reinterpret_cast<T*>(pool + off);
  off += count * sizeof(T);
  if (off > cap) ovf = true;
  return p;
}

template <class T, bool WG>
__global__ void __launch_bounds__(256, FA_FOREST_MINB) k_forest_dev(DevArgs<T, WG> A) {
  cg::grid_group grid = cg::this_grid();
  const uint32_t tid = (uint32_t)grid.thread_rank();
  const uint32_t nth = (uint32_t)grid.size();
  // a one-CTA grid (small graphs) synchronises with the CTA barrier
  const bool one_cta = gridDim.x == 1;
  auto sync_all = [&]() {
    if (one_cta) __syncthreads();
    else grid.sync();
  };
  // grid-stride loops in which every thread runs the same trip count (the
  // warp-collective appends need whole warps)
  auto trips = [&](uint32_t n) { return (n + nth - 1) / nth; };
  uint32_t* C = A.ctr;
  uint32_t n = A.n_dev ? min(__ldcg(A.n_dev), A.n0) : A.n0;
  const uint32_t* parent = A.parent0;
  T* val = A.val0;
  const T* wv = A.wv0;
  size_t off = 0;
  bool ovf = false;
  int level = 0;
  uint32_t nlevels = 0, njump = 0, nwalk = 0;  // statistics (uniform across threads)
  for (;;) {
    // ---------------- wide phase of this level
    if (tid == 0) {
      for (int i = 0; i < 16; ++i) C[i] = 0u;
    }
    for (uint32_t v = tid; v < n; v += nth) {
      A.cnt[v] = 0u;
      A.done[v] = 0u;
    }
    sync_all();
    for (uint32_t v = tid; v < n; v += nth) {
      const uint32_t p = parent[v];
      if (p != kNone) atomicAdd(&A.cnt[p], 1u);
    }
    sync_all();
    for (uint32_t t = 0, v = tid; t < trips(n); ++t, v += nth) {
      const uint32_t c = v < n ? ld(&A.cnt[v]) : 1u;
      if (v < n) A.one[v] = c == 1u;
      append(c == 0u, v, A.fa, &C[C_F + 0]);
    }
    sync_all();
    // rounds of capped walks ("the last arrival continues"); round r reads
    // the frontier count in slot r%3, appends to slot (r+1)%3 and zeroes
    // slot (r+2)%3 (read two barriers ago)
    uint32_t* cur = A.fa;
    uint32_t* nxt = A.fb;
    int r = 0;
    uint32_t nf = ld(&C[C_F + 0]);
    unsigned long long remaining = n;
    bool contract = false;
    while (nf > 0) {
      if ((unsigned long long)nf * (r > 0 ? kDevContractRatio : kDevLeafRatio) < remaining) {
        contract = true;
        break;
      }
      unsigned long long ret = 0;
      for (uint32_t t = 0, i = tid; t < trips(nf); ++t, i += nth) {
        bool push = false;
        uint32_t pnode = kNone;
        if (i < nf) {
          uint32_t v = cur[i];
          T s = __ldcg(&val[v]);
          uint32_t p = parent[v];
          for (int steps = 0;; ++steps) {
            A.done[v] = 1u;
            ++ret;
            if (p == kNone) break;
            // p's data is loaded in one round: with a single child (v) its
            // value is final once v's is added -- no atomics, one L2 round
            // trip per step along chains
            const bool one = __ldcg(&A.one[p]) != 0;
            const T vp = __ldcg(&val[p]);
            const uint32_t pp = parent[p];
            const T add = WG ? wv[v] * s : s;
            if (one) {
              s = vp + add;
              val[p] = s;
              if (steps + 1 >= A.cap) {
                A.cnt[p] = 0u;  // ready: no pending child
                push = true;
                pnode = p;
                break;
              }
            } else {
              atomic_add(&val[p], add);
              cuda::atomic_ref<uint32_t, cuda::thread_scope_device> cp(A.cnt[p]);
              if (cp.fetch_sub(1u, cuda::memory_order_acq_rel) != 1u) break;
              if (steps + 1 >= A.cap) {
                push = true;
                pnode = p;
                break;
              }
              s = __ldcg(&val[p]);
            }
            v = p;
            p = pp;
          }
        }
        append(push, pnode, nxt, &C[C_F + (r + 1) % 3]);
      }
      for (int o = 16; o; o >>= 1) ret += __shfl_xor_sync(0xFFFFFFFFu, ret, o);
      if ((threadIdx.x & 31) == 0 && ret) atomicAdd(reinterpret_cast<unsigned long long*>(&C[C_RET]), ret);
      if (tid == 0) C[C_F + (r + 2) % 3] = 0u;
      sync_all();
      ++r;
      ++nwalk;
      nf = ld(&C[C_F + r % 3]);
      remaining = (unsigned long long)n - ld64(&C[C_RET]);
      uint32_t* tmp = cur;
      cur = nxt;
      nxt = tmp;
    }
    if (!contract) {
      if (remaining != 0 && tid == 0) atomicOr(A.status, ST_CYCLE);  // some node never became ready
      break;
    }
    if (level + 1 >= kDevMaxLevels) {
      if (tid == 0) atomicOr(A.status, ST_CYCLE);
      break;
    }
    // ---------------- contraction of the residual forest (nodes not done)
    const uint32_t mcap = (uint32_t)remaining;
    DevLevel<T> L{};
    L.R = carve<uint32_t>(A.pool, off, mcap, A.pool_bytes, ovf);
    uint32_t* lpar = carve<uint32_t>(A.pool, off, mcap, A.pool_bytes, ovf);
    T* lval = carve<T>(A.pool, off, mcap, A.pool_bytes, ovf);
    uint32_t* lpc = carve<uint32_t>(A.pool, off, mcap, A.pool_bytes, ovf);
    uint32_t* up = carve<uint32_t>(A.pool, off, mcap, A.pool_bytes, ovf);
    uint32_t* nxa = carve<uint32_t>(A.pool, off, mcap, A.pool_bytes, ovf);
    uint32_t* nxb = carve<uint32_t>(A.pool, off, mcap, A.pool_bytes, ovf);
    T* aca = carve<T>(A.pool, off, mcap, A.pool_bytes, ovf);
    T* acb = carve<T>(A.pool, off, mcap, A.pool_bytes, ovf);
    T* lw = WG ? carve<T>(A.pool, off, mcap, A.pool_bytes, ovf) : nullptr;
    T* mua = WG ? carve<T>(A.pool, off, mcap, A.pool_bytes, ovf) : nullptr;
    T* mub = WG ? carve<T>(A.pool, off, mcap, A.pool_bytes, ovf) : nullptr;
    L.sid = carve<uint32_t>(A.pool, off, mcap, A.pool_bytes, ovf);
    L.sval = carve<T>(A.pool, off, mcap, A.pool_bytes, ovf);
    uint32_t* spar = carve<uint32_t>(A.pool, off, mcap, A.pool_bytes, ovf);
    T* sw = WG ? carve<T>(A.pool, off, mcap, A.pool_bytes, ovf) : nullptr;
    if (ovf) {  // the host falls back to forest.cu
      if (tid == 0) {
        C[C_OVF] = 1u;
        if (A.stats_out) atomicOr(A.status, ST_RETRY);
      }
      break;
    }
    for (uint32_t t = 0, v = tid; t < trips(n); ++t, v += nth) {
      const bool keep = v < n && !A.done[v];
      const unsigned mask = __ballot_sync(0xFFFFFFFFu, keep);
      if (!mask) continue;
      const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
      uint32_t b0 = 0;
      if (lane == leader) b0 = atomicAdd(&C[C_M], (uint32_t)__popc(mask));
      b0 = __shfl_sync(0xFFFFFFFFu, b0, leader);
      if (keep) {
        const uint32_t q = b0 + __popc(mask & ((1u << lane) - 1));
        L.R[q] = v;
        A.rid[v] = q;
      }
    }
    sync_all();
    const uint32_t m = ld(&C[C_M]);
    L.m = m;
    L.val = val;
    for (uint32_t q = tid; q < m; q += nth) {
      const uint32_t v = L.R[q];
      if (WG) lw[q] = wv[v];
      const uint32_t p = parent[v];
      lpar[q] = p == kNone ? kNone : A.rid[p];
      lval[q] = __ldcg(&val[v]);
      lpc[q] = __ldcg(&A.cnt[v]);
      up[q] = kNone;
    }
    sync_all();
    for (uint32_t q = tid; q < m; q += nth) {
      const uint32_t pq = lpar[q];
      if (pq != kNone && lpc[pq] == 1u) up[pq] = q;  // the unique pending child of a chain node
    }
    sync_all();
    for (uint32_t q = tid; q < m; q += nth) {
      const bool start = lpc[q] != 1u;
      nxa[q] = start ? q : up[q];
      aca[q] = start ? (T)0 : lval[q];
      if (WG) mua[q] = start ? (T)1 : lw[up[q]];
    }
    sync_all();
    // pointer jumping along the unique-pending-child links
    for (int j = 0;; ++j) {
      bool ch = false;
      for (uint32_t q = tid; q < m; q += nth) {
        const uint32_t n1 = nxa[q];
        if (lpc[n1] != 1u) {
          nxb[q] = n1;
          acb[q] = aca[q];
          if (WG) mub[q] = mua[q];
        } else {
          nxb[q] = nxa[n1];
          if (WG) {
            acb[q] = aca[q] + mua[q] * aca[n1];
            mub[q] = mua[q] * mua[n1];
          } else {
            acb[q] = aca[q] + aca[n1];
          }
          ch = true;
        }
      }
      if (__syncthreads_or(ch) && threadIdx.x == 0) atomicOr(&C[C_CH + j % 3], 1u);
      // slot (j+1)%3 was last read after the barrier before the previous
      // round: zeroing it now cannot race a read; round j+1 sets it
      if (tid == 0) C[C_CH + (j + 1) % 3] = 0u;
      sync_all();
      {
        uint32_t* t1 = nxa;
        nxa = nxb;
        nxb = t1;
        T* t2 = aca;
        aca = acb;
        acb = t2;
        if (WG) {
          T* t3 = mua;
          mua = mub;
          mub = t3;
        }
      }
      ++njump;
      if (!ld(&C[C_CH + j % 3])) break;
      if (j + 1 > kDevMaxJump) {
        if (tid == 0) atomicOr(A.status, ST_CYCLE);
        break;
      }
    }
    L.nxt = nxa;
    L.acc = aca;
    L.mul = mua;
    // segment starts -> dense ids; their forest
    for (uint32_t t = 0, q = tid; t < trips(m); ++t, q += nth) {
      const bool start = q < m && lpc[q] != 1u;
      const unsigned mask = __ballot_sync(0xFFFFFFFFu, start);
      if (!mask) continue;
      const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
      uint32_t b0 = 0;
      if (lane == leader) b0 = atomicAdd(&C[C_MS], (uint32_t)__popc(mask));
      b0 = __shfl_sync(0xFFFFFFFFu, b0, leader);
      if (start) {
        const uint32_t s = b0 + __popc(mask & ((1u << lane) - 1));
        L.sid[q] = s;
        L.sval[s] = lval[q];
        spar[s] = kNone;
        if (WG) sw[s] = (T)0;
      }
    }
    sync_all();
    for (uint32_t q = tid; q < m; q += nth) {
      const uint32_t pq = lpar[q];
      if (pq != kNone && lpc[pq] == 1u) continue;  // not a segment end
      const uint32_t s = L.sid[nxa[q]];
      if (pq == kNone) {
        spar[s] = kNone;
      } else {
        spar[s] = L.sid[pq];
        if (WG) {
          sw[s] = lw[q] * mua[q];
          atomic_add(&L.sval[L.sid[pq]], lw[q] * aca[q]);
        } else {
          atomic_add(&L.sval[L.sid[pq]], aca[q]);
        }
      }
    }
    sync_all();
    const uint32_t ms = ld(&C[C_MS]);
    if (ms >= m) {  // no chain node in a thin residual: a cycle
      if (tid == 0) atomicOr(A.status, ST_CYCLE);
      break;
    }
    if (tid == 0) A.lv[level] = L;
    // descend: the segment forest is the next level's forest
    ++level;
    ++nlevels;
    n = ms;
    parent = spar;
    val = L.sval;
    wv = WG ? sw : nullptr;
    sync_all();  // every thread has read the level's counters before they are reset
  }
  if (tid == 0) {
    C[C_STATS] = nlevels;
    C[C_STATS + 1] = njump;
    C[C_STATS + 2] = nwalk;
    if (A.stats_out) {
      A.stats_out[0] = nlevels;
      A.stats_out[1] = njump;
      A.stats_out[2] = nwalk;
    }
  }
  sync_all();
  // ---------------- expand, deepest level first
  while (level > 0) {
    --level;
    const DevLevel<T> L = A.lv[level];
    for (uint32_t q = tid; q < L.m; q += nth) {
      const T sv = L.sval[L.sid[L.nxt[q]]];
      L.val[L.R[q]] = WG ? L.acc[q] + L.mul[q] * sv : sv + L.acc[q];
    }
    sync_all();
  }
}

// the root of every node (pointer jumping, forest.cu's k_root_jump rounds)
// as one cooperative launch: the convergence test after each round is read
// by every thread after the barrier (rotating flag slots as above), so no
// host read between rounds.  The result ends in ra.
__global__ void __launch_bounds__(256) k_roots_dev(uint32_t n, const uint32_t* __restrict__ parent, uint32_t* ra,
                                                   uint32_t* rb, uint32_t* flags, uint32_t* status) {
  cg::grid_group grid = cg::this_grid();
  const uint32_t tid = (uint32_t)grid.thread_rank();
  const uint32_t nth = (uint32_t)grid.size();
  for (uint32_t v = tid; v < n; v += nth) {
    const uint32_t p = parent[v];
    ra[v] = p == kNone ? v : p;
  }
  grid.sync();
  uint32_t* a = ra;
  uint32_t* b = rb;
  for (int j = 0;; ++j) {
    bool ch = false;
    for (uint32_t v = tid; v < n; v += nth) {
      const uint32_t x = ld(&a[v]), y = ld(&a[x]);
      b[v] = y;
      ch |= x != y;
    }
    if (__syncthreads_or(ch) && threadIdx.x == 0) atomicOr(&flags[j % 3], 1u);
    if (tid == 0) flags[(j + 1) % 3] = 0u;  // last read two barriers ago
    grid.sync();
    uint32_t* t = a;
    a = b;
    b = t;
    if (!ld(&flags[j % 3])) break;
    if (j + 1 > kDevMaxJump) {
      if (tid == 0) atomicOr(status, ST_CYCLE);
      break;
    }
  }
  if (a != ra)
    for (uint32_t v = tid; v < n; v += nth) ra[v] = a[v];
}

template <class T, bool WG>
cudaError_t solve_dev(Runtime& rt, uint32_t n, const uint32_t* parent, T* val, const T* wv, bool& done) {
  done = false;
  if (n == 0) {
    done = true;
    return cudaSuccess;
  }
  int dev = 0, sms = 0, coop = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop) return cudaSuccess;  // not done: forest.cu solves it
  auto k = k_forest_dev<T, WG>;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, 0) != cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    return cudaSuccess;
  }
  cudaStream_t st = rt.st;
  DevArgs<T, WG> a{};
  a.n0 = n;
  a.parent0 = parent;
  a.val0 = val;
  a.wv0 = wv;
  a.cnt = rt.alloc<uint32_t>(n);
  a.done = rt.alloc<uint8_t>(n);
  a.one = rt.alloc<uint8_t>(n);
  a.fa = rt.alloc<uint32_t>(n);
  a.fb = rt.alloc<uint32_t>(n);
  a.rid = rt.alloc<uint32_t>(n);
  a.ctr = rt.alloc<uint32_t>(64);
  // level states: the residual of level 0 is at most n nodes, each deeper
  // level at most the previous one's segments
  const size_t per = 4 * 7 + sizeof(T) * (WG ? 8 : 4) + 64;
  a.pool_bytes = per * ((size_t)n + 4096) + (size_t)n * per / 2;
  a.pool = rt.alloc<uint8_t>(a.pool_bytes);
  a.lv = rt.alloc<DevLevel<T>>(kDevMaxLevels);
  a.status = rt.d_status;
  a.cap = rt.walk_cap > 0 ? rt.walk_cap : 1;  // walk cap 0 ("peel only"): one step per round
  if (rt.err) return rt.err;
  cudaMemsetAsync(a.ctr, 0, 64 * sizeof(uint32_t), st);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * per_sm, ((int64_t)n + 255) / 256));
  void* args[] = {&a};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)k, grid, 256, args, 0, st);
  ++rt.launches;
  if (e != cudaSuccess) {
    cudaGetLastError();
    for (void* p : {(void*)a.cnt, (void*)a.done, (void*)a.one, (void*)a.fa, (void*)a.fb, (void*)a.rid, (void*)a.ctr,
                    (void*)a.pool, (void*)a.lv})
      rt.free(p);
    return cudaSuccess;  // not done: forest.cu solves it
  }
  // the pool-overflow flag: read back only to decide a fallback (one small
  // copy, after the solve; never set in practice)
  e = cudaMemcpyAsync(rt.h_cnt + 12, a.ctr + C_OVF, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  for (void* p : {(void*)a.cnt, (void*)a.done, (void*)a.one, (void*)a.fa, (void*)a.fb, (void*)a.rid, (void*)a.ctr,
                  (void*)a.pool, (void*)a.lv})
    rt.free(p);
  if (e != cudaSuccess) return e;
  done = rt.h_cnt[12] == 0u;
  if (done) {
    rt.contract_levels += rt.h_cnt[13];
    rt.jump_rounds += rt.h_cnt[14];
    rt.peel_rounds += rt.h_cnt[15];
  }
  return cudaSuccess;
}

// the same solve without any host read: the node count is read on the device,
// scratch is sized for the bound n_max, statistics go to stats_out, and a
// scratch overflow raises ST_RETRY in the status word instead of a fallback
template <class T>
cudaError_t solve_dev_async(Runtime& rt, uint32_t n_max, const uint32_t* n_dev, const uint32_t* parent, T* val,
                            uint32_t* stats_out) {
  if (n_max == 0) return cudaSuccess;
  int dev = 0, sms = 0, coop = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  auto k = k_forest_dev<T, false>;
  if (!coop || cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, 0) != cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    return cudaErrorNotSupported;
  }
  cudaStream_t st = rt.st;
  DevArgs<T, false> a{};
  a.n0 = n_max;
  a.n_dev = n_dev;
  a.stats_out = stats_out;
  a.parent0 = parent;
  a.val0 = val;
  a.cnt = rt.alloc<uint32_t>(n_max);
  a.done = rt.alloc<uint8_t>(n_max);
  a.one = rt.alloc<uint8_t>(n_max);
  a.fa = rt.alloc<uint32_t>(n_max);
  a.fb = rt.alloc<uint32_t>(n_max);
  a.rid = rt.alloc<uint32_t>(n_max);
  a.ctr = rt.alloc<uint32_t>(64);
  const size_t per = 4 * 7 + sizeof(T) * 4 + 64;
  a.pool_bytes = per * ((size_t)n_max + 4096) + (size_t)n_max * per / 2;
  a.pool = rt.alloc<uint8_t>(a.pool_bytes);
  a.lv = rt.alloc<DevLevel<T>>(kDevMaxLevels);
  a.status = rt.d_status;
  a.cap = rt.walk_cap > 0 ? rt.walk_cap : 1;
  if (rt.err) return rt.err;
  cudaMemsetAsync(a.ctr, 0, 64 * sizeof(uint32_t), st);
  // a small graph gets a small grid: its barriers are cheaper (one CTA per
  // 256 nodes; a single CTA synchronises with its own barrier)
  if (FA_FOREST_PER_SM > 0 && per_sm > FA_FOREST_PER_SM) per_sm = FA_FOREST_PER_SM;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * per_sm, ((int64_t)n_max + 255) / 256));
  void* args[] = {&a};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)k, grid, 256, args, 0, st);
  ++rt.launches;
  for (void* p : {(void*)a.cnt, (void*)a.done, (void*)a.one, (void*)a.fa, (void*)a.fb, (void*)a.rid, (void*)a.ctr, (void*)a.pool,
                  (void*)a.lv})
    rt.free(p);
  return e;
}

}  // namespace

template <class T>
cudaError_t forest_solve_device_async(Runtime& rt, uint32_t n_max, const uint32_t* n_dev, const uint32_t* parent,
                                      T* val, uint32_t* stats_out) {
  return solve_dev_async<T>(rt, n_max, n_dev, parent, val, stats_out);
}
template cudaError_t forest_solve_device_async<uint32_t>(Runtime&, uint32_t, const uint32_t*, const uint32_t*,
                                                         uint32_t*, uint32_t*);
template cudaError_t forest_solve_device_async<unsigned long long>(Runtime&, uint32_t, const uint32_t*,
                                                                   const uint32_t*, unsigned long long*, uint32_t*);
template cudaError_t forest_solve_device_async<double>(Runtime&, uint32_t, const uint32_t*, const uint32_t*, double*,
                                                       uint32_t*);

cudaError_t forest_roots_device(Runtime& rt, uint32_t n, const uint32_t* parent, uint32_t* root) {
  if (n == 0) return cudaSuccess;
  int dev = 0, sms = 0, coop = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop || cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_roots_dev, 256, 0) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    return cudaErrorNotSupported;
  }
  cudaStream_t st = rt.st;
  uint32_t* tmp = rt.alloc<uint32_t>(n);
  uint32_t* flags = rt.alloc<uint32_t>(4);
  if (rt.err) return rt.err;
  cudaMemsetAsync(flags, 0, 4 * sizeof(uint32_t), st);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * per_sm, ((int64_t)n + 255) / 256));
  uint32_t* status = rt.d_status;
  void* args[] = {&n, &parent, &root, &tmp, &flags, &status};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_roots_dev, grid, 256, args, 0, st);
  ++rt.launches;
  rt.free(tmp);
  rt.free(flags);
  return e;
}

template <class T>
cudaError_t forest_solve_device(Runtime& rt, uint32_t n, const uint32_t* parent, T* val, bool& done) {
  return solve_dev<T, false>(rt, n, parent, val, nullptr, done);
}
cudaError_t forest_solve_weighted_device(Runtime& rt, uint32_t n, const uint32_t* parent, const double* wv,
                                         double* val, bool& done) {
  return solve_dev<double, true>(rt, n, parent, val, wv, done);
}
template cudaError_t forest_solve_device<uint32_t>(Runtime&, uint32_t, const uint32_t*, uint32_t*, bool&);
template cudaError_t forest_solve_device<unsigned long long>(Runtime&, uint32_t, const uint32_t*,
                                                             unsigned long long*, bool&);
template cudaError_t forest_solve_device<double>(Runtime&, uint32_t, const uint32_t*, double*, bool&);

}  // namespace fa
