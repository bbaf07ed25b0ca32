// forest.cu -- accumulation on an explicit forest (the perimeter / block-exit
// graphs), S(v) = val(v) + sum_{children c} S(c).
//
// The paper solves its global flow graph "using the same strategy described
// in Algorithm 1": dependency counts and a queue of ready nodes.  A
// level-synchronous version of that (one kernel per round, warp-aggregated
// atomics) is efficient while the ready frontier is wide.  Deep graphs
// (rivers crossing hundreds of blocks, the serpentine of config 2) make the
// frontier "long and thin", so once it falls below remaining/8 the residual
// forest is contracted instead:
//   * every residual node with exactly one pending child is a chain node; a
//     node with 0 or >= 2 pending children starts a segment;
//   * pointer jumping along the unique-pending-child links gives every node
//     its segment start st(v) and the prefix pre(v) of values from st(v)
//     (exclusive) down to v (inclusive): S(v) = S(st(v)) + pre(v);
//   * the segment starts form a smaller forest (every internal node has >= 2
//     children), solved recursively; then S is expanded back.
// This is rake (peel) + compress (chain jumping) tree contraction, O(log)
// phases; each phase is a handful of grid-stride kernels.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cuda/atomic>

#include "forest.cuh"

#ifndef FA_WALK_FAST
#define FA_WALK_FAST 1  // walks take single-child parents without atomics
#endif

namespace fa {

namespace {

__global__ void k_count_children(uint32_t n, const uint32_t* __restrict__ parent, uint32_t* cnt) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint32_t p = parent[v];
    if (p != kNone) atomicAdd(&cnt[p], 1u);
  }
}

// CTA-aggregated append (every thread of the CTA calls it): one global
// atomic per CTA instead of one per warp -- the frontier of the first round
// holds most nodes, and per-warp atomics on one counter serialise in L2
template <int NT>
__device__ __forceinline__ void cta_append(bool pred, uint32_t v, uint32_t* list, uint32_t* count,
                                           uint32_t* s_tmp /* NT/32 + 1 words of shared memory */) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned mask = __ballot_sync(0xFFFFFFFFu, pred);
  if (lane == 0) s_tmp[w] = (uint32_t)__popc(mask);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t tot = 0;
    for (int i = 0; i < NT / 32; ++i) {
      const uint32_t c = s_tmp[i];
      s_tmp[i] = tot;
      tot += c;
    }
    s_tmp[NT / 32] = tot ? atomicAdd(count, tot) : 0u;
  }
  __syncthreads();
  if (pred) list[s_tmp[NT / 32] + s_tmp[w] + (uint32_t)__popc(mask & ((1u << lane) - 1u))] = v;
  __syncthreads();  // s_tmp is reused by the next call
}

// frontier = {v : cnt[v] == 0}; done[v] = 0.  All threads iterate uniformly.
// one[v]: v has exactly one child (k_walk's fast path).
__global__ void __launch_bounds__(256) k_init_frontier(uint32_t n, const uint32_t* __restrict__ cnt, uint8_t* done,
                                                       uint8_t* one, uint32_t* front, uint32_t* fcount) {
  __shared__ uint32_t s_tmp[256 / 32 + 1];
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x; base < n; base += stride) {
    const uint32_t v = base + threadIdx.x;
    const uint32_t c = v < n ? cnt[v] : 1u;
    if (v < n) {
      done[v] = 0;
      one[v] = c == 1u;
    }
    cta_append<256>(c == 0u, v, front, fcount, s_tmp);
  }
}

// One level-synchronous peel round (Alg. 1's queue loop over the forest)
// with the frontier size read on the device: rounds are
// launched back to back without a host round trip.  Counters rotate over
// three slots: round r reads c[r%3], appends into c[(r+1)%3] (zeroed by round
// r-1) and zeroes c[(r+2)%3] for round r+1; `retired` accumulates the sizes.
template <class T, bool WG = false>
__global__ void k_peel_dev(const uint32_t* __restrict__ front, const uint32_t* __restrict__ nf_in,
                           const uint32_t* __restrict__ parent, T* val, uint32_t* cnt, uint8_t* done,
                           uint32_t* next, uint32_t* nf_out, uint32_t* nf_clear,
                           unsigned long long* retired, const T* __restrict__ wv) {
  const uint32_t nf = *nf_in;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *nf_clear = 0u;
    *retired += nf;
  }
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x; base < nf; base += stride) {
    const uint32_t i = base + threadIdx.x;
    bool push = false;
    uint32_t p = kNone;
    if (i < nf) {
      const uint32_t v = front[i];
      done[v] = 1;
      p = parent[v];
      if (p != kNone) {
        atomic_add(&val[p], WG ? wv[v] * val[v] : val[v]);  // absorption: edge weight
        push = atomicSub(&cnt[p], 1u) == 1u;
      }
    }
    warp_append(push, p, next, nf_out);
  }
}

// Walks on the global forest ("last arrival continues"): each ready node adds
// its finished sum into its parent; the thread whose decrement retires the
// parent's last pending child continues from the parent.  One launch replaces
// the wide rounds of level-synchronous peeling; a walk stops after `cap`
// steps and re-queues the ready node, leaving deep chains to contraction.
template <class T, bool WG = false>
__global__ void k_walk(const uint32_t* __restrict__ front, const uint32_t* __restrict__ nf_dev,
                       const uint32_t* __restrict__ parent, T* val, uint32_t* cnt, uint8_t* done,
                       const uint8_t* __restrict__ one, uint32_t* next, uint32_t* ncount, uint32_t* nretired, int cap,
                       const T* __restrict__ wv) {
  const uint32_t nf = *nf_dev;  // frontier size read on the device: no host round trip before the launch
  const uint32_t stride = gridDim.x * blockDim.x;
  uint32_t retired = 0;
  for (uint32_t base = blockIdx.x * blockDim.x; base < nf; base += stride) {
    const uint32_t i = base + threadIdx.x;
    bool push = false;
    uint32_t pnode = kNone;
    if (i < nf) {
      uint32_t v = front[i];
      T s = __ldcg(&val[v]);
      uint32_t p = parent[v];
      for (int steps = 0;; ++steps) {
        done[v] = 1;
        ++retired;
        if (p == kNone) break;
        // p's flag, value and parent in one round of loads: with a single
        // child (v) p is final once v's sum is added -- no atomics, one L2
        // round trip per step along chains
        const bool single = FA_WALK_FAST && one[p] != 0;
        const T vp = __ldcg(&val[p]);
        const uint32_t pp = parent[p];
        const T add = WG ? wv[v] * s : s;
        if (single) {
          s = vp + add;
          val[p] = s;
          if (steps + 1 >= cap) {
            cnt[p] = 0u;  // ready: no pending child
            push = true;
            pnode = p;
            break;
          }
        } else {
          atomic_add(&val[p], add);
          // acq_rel decrement: our contribution is released before it, and the
          // last arrival acquires every other child's contribution
          cuda::atomic_ref<uint32_t, cuda::thread_scope_device> cp(cnt[p]);
          if (cp.fetch_sub(1u, cuda::memory_order_acq_rel) != 1u) break;
          if (steps + 1 >= cap) {
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
    warp_append(push, pnode, next, ncount);
  }
  // one global atomic per CTA (the retired count is a single counter)
  __shared__ uint32_t s_ret;
  if (threadIdx.x == 0) s_ret = 0u;
  __syncthreads();
  for (int o = 16; o; o >>= 1) retired += __shfl_xor_sync(0xFFFFFFFFu, retired, o);
  if ((threadIdx.x & 31) == 0 && retired) atomicAdd(&s_ret, retired);
  __syncthreads();
  if (threadIdx.x == 0 && s_ret) atomicAdd(nretired, s_ret);
}

__global__ void k_compact_residual(uint32_t n, const uint8_t* __restrict__ done, uint32_t* R,
                                   uint32_t* mcount, uint32_t* rid) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x; base < n; base += stride) {
    const uint32_t v = base + threadIdx.x;
    const bool keep = v < n && !done[v];
    // rid assigned after the append: recompute position via a second pass is
    // avoided by writing rid inside warp_append's ordering below
    const unsigned mask = __ballot_sync(0xFFFFFFFFu, keep);
    if (!mask) continue;
    const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
    uint32_t b0 = 0;
    if (lane == leader) b0 = atomicAdd(mcount, (uint32_t)__popc(mask));
    b0 = __shfl_sync(0xFFFFFFFFu, b0, leader);
    if (keep) {
      const uint32_t r = b0 + __popc(mask & ((1u << lane) - 1));
      R[r] = v;
      rid[v] = r;
    }
  }
}

template <class T, bool WG = false>
__global__ void k_build_local(uint32_t m, const uint32_t* __restrict__ R,
                              const uint32_t* __restrict__ parent, const T* __restrict__ val,
                              const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ rid,
                              uint32_t* lpar, T* lval, uint32_t* lpc, uint32_t* up,
                              const T* __restrict__ wv, T* lw) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x) {
    const uint32_t v = R[r];
    if (WG) lw[r] = wv[v];  // weight of r's edge to its parent
    const uint32_t p = parent[v];
    lpar[r] = p == kNone ? kNone : rid[p];
    lval[r] = val[v];
    lpc[r] = cnt[v];
    up[r] = kNone;
  }
}

__global__ void k_set_up(uint32_t m, const uint32_t* __restrict__ lpar, const uint32_t* __restrict__ lpc,
                         uint32_t* up) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x) {
    const uint32_t q = lpar[r];
    if (q != kNone && lpc[q] == 1u) up[q] = r;
  }
}

// weighted (absorption): S(r) = acc(r) + mul(r) S(nxt(r)); a chain node's
// single pending child c contributes w(c) S(c)
template <class T, bool WG = false>
__global__ void k_jump_init(uint32_t m, const uint32_t* __restrict__ lpc, const uint32_t* __restrict__ up,
                            const T* __restrict__ lval, uint32_t* nxt, T* acc, const T* __restrict__ lw, T* mul) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x) {
    const bool start = lpc[r] != 1u;
    nxt[r] = start ? r : up[r];
    acc[r] = start ? (T)0 : lval[r];
    if (WG) mul[r] = start ? (T)1 : lw[up[r]];
  }
}

template <class T, bool WG = false>
__global__ void k_jump(uint32_t m, const uint32_t* __restrict__ lpc, const uint32_t* __restrict__ nxt_in,
                       const T* __restrict__ acc_in, uint32_t* nxt_out, T* acc_out, uint32_t* changed,
                       const T* __restrict__ mul_in, T* mul_out) {
  bool ch = false;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x) {
    const uint32_t n1 = nxt_in[r];
    if (lpc[n1] != 1u) {  // reached a segment start
      nxt_out[r] = n1;
      acc_out[r] = acc_in[r];
      if (WG) mul_out[r] = mul_in[r];
    } else {
      nxt_out[r] = nxt_in[n1];
      if (WG) {
        acc_out[r] = acc_in[r] + mul_in[r] * acc_in[n1];
        mul_out[r] = mul_in[r] * mul_in[n1];
      } else {
        acc_out[r] = acc_in[r] + acc_in[n1];
      }
      ch = true;
    }
  }
  if (__syncthreads_or(ch) && threadIdx.x == 0) atomicOr(changed, 1u);
}

// starts -> dense segment ids; sval = own value, spar = kNone
template <class T>
__global__ void k_seg_ids(uint32_t m, const uint32_t* __restrict__ lpc, const T* __restrict__ lval,
                          uint32_t* sid, uint32_t* scount, T* sval, uint32_t* spar) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x; base < m; base += stride) {
    const uint32_t r = base + threadIdx.x;
    const bool start = r < m && lpc[r] != 1u;
    const unsigned mask = __ballot_sync(0xFFFFFFFFu, start);
    if (!mask) continue;
    const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
    uint32_t b0 = 0;
    if (lane == leader) b0 = atomicAdd(scount, (uint32_t)__popc(mask));
    b0 = __shfl_sync(0xFFFFFFFFu, b0, leader);
    if (start) {
      const uint32_t s = b0 + __popc(mask & ((1u << lane) - 1));
      sid[r] = s;
      sval[s] = lval[r];
      spar[s] = kNone;
    }
  }
}

// every segment end r (parent is a junction or none) links its segment start
// to the junction and hands the junction its chain prefix pre(r)
template <class T, bool WG = false>
__global__ void k_seg_build(uint32_t m, const uint32_t* __restrict__ lpar, const uint32_t* __restrict__ lpc,
                            const uint32_t* __restrict__ nxt, const T* __restrict__ acc,
                            const uint32_t* __restrict__ sid, uint32_t* spar, T* sval,
                            const T* __restrict__ lw, const T* __restrict__ mul, T* sw) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x) {
    const uint32_t q = lpar[r];
    if (q != kNone && lpc[q] == 1u) continue;  // not an end
    const uint32_t s = sid[nxt[r]];
    if (q == kNone) {
      spar[s] = kNone;
    } else {
      spar[s] = sid[q];
      if (WG) {
        // S(q) += w(r) S(r) = w(r) acc(r) + w(r) mul(r) S(start): the segment edge weight
        sw[s] = lw[r] * mul[r];
        atomic_add(&sval[sid[q]], lw[r] * acc[r]);
      } else {
        atomic_add(&sval[sid[q]], acc[r]);
      }
    }
  }
}

template <class T, bool WG = false>
__global__ void k_expand(uint32_t m, const uint32_t* __restrict__ R, const uint32_t* __restrict__ nxt,
                         const T* __restrict__ acc, const uint32_t* __restrict__ sid,
                         const T* __restrict__ sval, T* val, const T* __restrict__ mul) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x)
    val[R[r]] = WG ? acc[r] + mul[r] * sval[sid[nxt[r]]] : sval[sid[nxt[r]]] + acc[r];
}

__global__ void k_set_flag(uint32_t* st, uint32_t f) { atomicOr(st, f); }

constexpr int kMaxLevels = 64;
constexpr int kPeelBatch = 4;  // peel rounds per host check
constexpr int kMaxJump = 40;
constexpr uint64_t kContractRatio = 8;  // contract once the frontier < remaining / 8
// walk cap (Runtime::walk_cap, FA_OPT_WALK_CAP): steps per walk before
// re-queueing (deep chains -> contraction); 0 = peel only.  128 vs 32: cfg3
// graph 1.54 vs 1.57 ms, 8 strips 29.9 vs 31.1 ms, cfg2 (one 16.7M chain) 1.04 vs 0.95 ms

// WG (absorption): edge weights wv (S(parent) += wv(v) S(v)); chains are
// contracted with affine (acc, mul) pairs instead of sums
template <class T, bool WG = false>
cudaError_t solve_level(Runtime& rt, uint32_t n, const uint32_t* parent, T* val, int level,
                        const T* wv = nullptr) {
  if (n == 0) return cudaSuccess;
  if (level > kMaxLevels) {
    k_set_flag<<<1, 1, 0, rt.st>>>(rt.d_status, ST_CYCLE);
    ++rt.launches;
    return cudaGetLastError();
  }
  cudaStream_t st = rt.st;
  uint32_t* cnt = rt.alloc<uint32_t>(n);
  uint8_t* done = rt.alloc<uint8_t>(n);
  uint8_t* one = rt.alloc<uint8_t>(n);
  uint32_t* fa_ = rt.alloc<uint32_t>(n);
  uint32_t* fb = rt.alloc<uint32_t>(n);
  uint32_t* ctr = rt.alloc<uint32_t>(4);
  if (rt.err) return rt.err;
  cudaMemsetAsync(cnt, 0, n * sizeof(uint32_t), st);
  cudaMemsetAsync(ctr, 0, 4 * sizeof(uint32_t), st);
  k_count_children<<<grid_for(n), 256, 0, st>>>(n, parent, cnt);
  ++rt.launches;
  k_init_frontier<<<grid_for(n), 256, 0, st>>>(n, cnt, done, one, fa_, ctr);
  ++rt.launches;
  uint32_t nf = 1;  // the frontier size stays on the device until after the walks
  uint64_t remaining = n;
  bool contracted = false;
  uint32_t* pc = nullptr;  // device frontier counters of the batched peel rounds
  const int cap = rt.walk_cap;
  if (cap <= 0) {
    rt.read(ctr, 1);
    nf = rt.h_cnt[0];
  } else {
    // bulk of the forest: one launch of capped walks from every leaf (a
    // grid for all n nodes; the walks read the frontier size themselves)
    cudaMemsetAsync(ctr + 1, 0, 2 * sizeof(uint32_t), st);
    k_walk<T, WG><<<grid_for(n), 256, 0, st>>>(fa_, ctr, parent, val, cnt, done, one, fb, ctr + 1, ctr + 2, cap, wv);
    ++rt.launches;
    ++rt.peel_rounds;
    std::swap(fa_, fb);
    cudaMemcpyAsync(ctr, ctr + 1, sizeof(uint32_t), cudaMemcpyDeviceToDevice, st);  // frontier size for the peel
    rt.read(ctr + 1, 2);
    nf = rt.h_cnt[0];
    remaining -= rt.h_cnt[1];
  }
  while (nf > 0 && !rt.err) {
    if ((uint64_t)nf * kContractRatio < remaining) {
      // ---------------- contract the residual forest
      contracted = true;
      ++rt.contract_levels;
      uint32_t* R = rt.alloc<uint32_t>(remaining);
      uint32_t* rid = rt.alloc<uint32_t>(n);
      cudaMemsetAsync(ctr + 1, 0, sizeof(uint32_t), st);
      k_compact_residual<<<grid_for(n), 256, 0, st>>>(n, done, R, ctr + 1, rid);
      ++rt.launches;
      const uint32_t m = (uint32_t)remaining;
      uint32_t* lpar = rt.alloc<uint32_t>(m);
      uint32_t* lpc = rt.alloc<uint32_t>(m);
      uint32_t* up = rt.alloc<uint32_t>(m);
      uint32_t* nxa = rt.alloc<uint32_t>(m);
      uint32_t* nxb = rt.alloc<uint32_t>(m);
      uint32_t* sid = rt.alloc<uint32_t>(m);
      T* lval = rt.alloc<T>(m);
      T* aca = rt.alloc<T>(m);
      T* acb = rt.alloc<T>(m);
      T* lw = WG ? rt.alloc<T>(m) : nullptr;
      T* mua = WG ? rt.alloc<T>(m) : nullptr;
      T* mub = WG ? rt.alloc<T>(m) : nullptr;
      if (rt.err) return rt.err;
      k_build_local<T, WG><<<grid_for(m), 256, 0, st>>>(m, R, parent, val, cnt, rid, lpar, lval, lpc, up, wv, lw);
      ++rt.launches;
      k_set_up<<<grid_for(m), 256, 0, st>>>(m, lpar, lpc, up);
      ++rt.launches;
      k_jump_init<T, WG><<<grid_for(m), 256, 0, st>>>(m, lpc, up, lval, nxa, aca, lw, mua);
      ++rt.launches;
      int rounds = 0;
      for (int batch = 8;; batch = 4) {
        // pointer jumping converges in ceil(log2(longest chain)) rounds; the
        // "changed" flag is read back after 8 rounds, then every 4 (extra
        // rounds are no-ops)
        cudaMemsetAsync(ctr + 2, 0, sizeof(uint32_t), st);
        for (int j = 0; j < batch; ++j) {
          k_jump<T, WG><<<grid_for(m), 256, 0, st>>>(m, lpc, nxa, aca, nxb, acb, ctr + 2, mua, mub);
          std::swap(nxa, nxb);
          std::swap(aca, acb);
          std::swap(mua, mub);
        }
        rt.launches += batch;
        rounds += batch;
        rt.jump_rounds += batch;
        rt.read(ctr + 2, 1);
        if (!rt.h_cnt[0] || rt.err) break;
        if (rounds > kMaxJump) {
          k_set_flag<<<1, 1, 0, st>>>(rt.d_status, ST_CYCLE);
          ++rt.launches;
          break;
        }
      }
      // segment forest over the starts
      cudaMemsetAsync(ctr + 3, 0, sizeof(uint32_t), st);
      T* sval = rt.alloc<T>(m);
      uint32_t* spar = rt.alloc<uint32_t>(m);
      T* sw = WG ? rt.alloc<T>(m) : nullptr;
      if (rt.err) return rt.err;
      if (WG) cudaMemsetAsync(sw, 0, m * sizeof(T), st);
      k_seg_ids<T><<<grid_for(m), 256, 0, st>>>(m, lpc, lval, sid, ctr + 3, sval, spar);
      ++rt.launches;
      k_seg_build<T, WG><<<grid_for(m), 256, 0, st>>>(m, lpar, lpc, nxa, aca, sid, spar, sval, lw, mua, sw);
      ++rt.launches;
      rt.read(ctr + 3, 1);
      const uint32_t ms = rt.h_cnt[0];
      if (rounds <= kMaxJump && ms < m) {
        solve_level<T, WG>(rt, ms, spar, sval, level + 1, sw);
      } else if (ms >= m) {
        // no chain node: cannot happen with a thin frontier unless cyclic
        k_set_flag<<<1, 1, 0, st>>>(rt.d_status, ST_CYCLE);
        ++rt.launches;
      }
      k_expand<T, WG><<<grid_for(m), 256, 0, st>>>(m, R, nxa, aca, sid, sval, val, mua);
      ++rt.launches;
      for (void* p : {(void*)R, (void*)rid, (void*)lpar, (void*)lpc, (void*)up, (void*)nxa,
                      (void*)nxb, (void*)sid, (void*)lval, (void*)aca, (void*)acb, (void*)sval,
                      (void*)spar, (void*)lw, (void*)mua, (void*)mub, (void*)sw})
        rt.free(p);
      remaining = 0;
      break;
    }
    // ---------------- kPeelBatch peel rounds (Alg. 1 queue loop, level-
    // synchronous), frontier sizes kept on the device; one read per batch
    if (!pc) {
      pc = rt.alloc<uint32_t>(8);  // [0..2] rotating frontier counters, [4..5] retired (u64)
      if (rt.err) return rt.err;
    }
    cudaMemsetAsync(pc, 0, 8 * sizeof(uint32_t), st);
    cudaMemcpyAsync(pc, ctr, sizeof(uint32_t), cudaMemcpyDeviceToDevice, st);  // c[0] = nf
    unsigned long long* retired = reinterpret_cast<unsigned long long*>(pc + 4);
    const unsigned grid = grid_for(nf);
    for (int r = 0; r < kPeelBatch; ++r) {
      k_peel_dev<T, WG><<<grid, 256, 0, st>>>(fa_, pc + r % 3, parent, val, cnt, done, fb, pc + (r + 1) % 3,
                                              pc + (r + 2) % 3, retired, wv);
      std::swap(fa_, fb);
    }
    rt.launches += kPeelBatch;
    rt.peel_rounds += kPeelBatch;
    cudaMemcpyAsync(ctr, pc + kPeelBatch % 3, sizeof(uint32_t), cudaMemcpyDeviceToDevice, st);
    rt.read(pc, 6);
    nf = rt.h_cnt[kPeelBatch % 3];
    unsigned long long ret = 0;
    memcpy(&ret, &rt.h_cnt[4], sizeof(ret));
    remaining -= ret;
  }
  rt.free(pc);
  if (!contracted && remaining != 0) k_set_flag<<<1, 1, 0, st>>>(rt.d_status, ST_CYCLE);
  rt.free(cnt);
  rt.free(done);
  rt.free(one);
  rt.free(fa_);
  rt.free(fb);
  rt.free(ctr);
  return rt.err ? rt.err : cudaGetLastError();
}

// ---------------------------------------------------------------- roots
__global__ void k_root_init(uint32_t n, const uint32_t* __restrict__ parent, uint32_t* r) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    r[v] = parent[v] == kNone ? v : parent[v];
}
__global__ void k_root_jump(uint32_t n, const uint32_t* __restrict__ in, uint32_t* out, uint32_t* changed) {
  bool ch = false;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint32_t a = in[v], b = in[a];
    out[v] = b;
    ch |= a != b;
  }
  if (__syncthreads_or(ch) && threadIdx.x == 0) atomicOr(changed, 1u);
}

}  // namespace

template <class T>
cudaError_t forest_solve(Runtime& rt, uint32_t n, const uint32_t* parent, T* val) {
  if (rt.use_device_solver(n)) {  // one cooperative launch, no host round trip (forest_dev.cu)
    bool done = false;
    const cudaError_t e = forest_solve_device<T>(rt, n, parent, val, done);
    if (e != cudaSuccess || done) return e;
  }
  return solve_level<T>(rt, n, parent, val, 0);
}
template cudaError_t forest_solve<uint32_t>(Runtime&, uint32_t, const uint32_t*, uint32_t*);
template cudaError_t forest_solve<unsigned long long>(Runtime&, uint32_t, const uint32_t*,
                                                      unsigned long long*);
template cudaError_t forest_solve<double>(Runtime&, uint32_t, const uint32_t*, double*);

cudaError_t forest_roots(Runtime& rt, uint32_t n, const uint32_t* parent, uint32_t* root) {
  if (n == 0) return cudaSuccess;
  {  // one cooperative launch when possible (no host read between rounds)
    const cudaError_t e = forest_roots_device(rt, n, parent, root);
    if (e != cudaErrorNotSupported) return e;
  }
  cudaStream_t st = rt.st;
  uint32_t* tmp = rt.alloc<uint32_t>(n);
  uint32_t* ctr = rt.alloc<uint32_t>(1);
  if (rt.err) return rt.err;
  k_root_init<<<grid_for(n), 256, 0, st>>>(n, parent, root);
  ++rt.launches;
  uint32_t* a = root;
  uint32_t* b = tmp;
  int rounds = 0;
  for (int batch = 8;; batch = 4) {
    // converged rounds are no-ops: 8 rounds (depth 256) before the first
    // host check, then a check every 4
    cudaMemsetAsync(ctr, 0, sizeof(uint32_t), st);
    for (int j = 0; j < batch; ++j) {
      k_root_jump<<<grid_for(n), 256, 0, st>>>(n, a, b, ctr);
      std::swap(a, b);
    }
    rt.launches += batch;
    rounds += batch;
    rt.read(ctr, 1);
    if (!rt.h_cnt[0] || rt.err) break;
    if (rounds > kMaxJump) {
      k_set_flag<<<1, 1, 0, st>>>(rt.d_status, ST_CYCLE);
      ++rt.launches;
      break;
    }
  }
  if (a != root) cudaMemcpyAsync(root, a, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st);
  rt.free(tmp);
  rt.free(ctr);
  return rt.err ? rt.err : cudaGetLastError();
}

// ---------------------------------------------------------------- weighted forest (absorption)
// S(v) = val(v) + sum_children wv(c) S(c): the same walk / peel / contract
// solver with edge weights (affine chain contraction)
cudaError_t forest_solve_weighted(Runtime& rt, uint32_t n, const uint32_t* parent, const double* wv, double* val) {
  if (rt.use_device_solver(n)) {
    bool done = false;
    const cudaError_t e = forest_solve_weighted_device(rt, n, parent, wv, val, done);
    if (e != cudaSuccess || done) return e;
  }
  return solve_level<double, true>(rt, n, parent, val, 0, wv);
}

// roots with path products (absorption): root(v) and prod(v) = the product of
// the edge weights wv on the path from v up to its root
namespace {
__global__ void k_root_init_w(uint32_t n, const uint32_t* __restrict__ parent, const double* __restrict__ wv,
                              uint32_t* r, double* pr) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const bool top = parent[v] == kNone;
    r[v] = top ? v : parent[v];
    pr[v] = top ? 1.0 : wv[v];
  }
}
__global__ void k_root_jump_w(uint32_t n, const uint32_t* __restrict__ in, const double* __restrict__ pin,
                              uint32_t* out, double* pout, uint32_t* changed) {
  bool ch = false;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint32_t a = in[v], b = in[a];
    out[v] = b;
    pout[v] = a == b ? pin[v] : pin[v] * pin[a];  // the root's own product is 1
    ch |= a != b;
  }
  if (__syncthreads_or(ch) && threadIdx.x == 0) atomicOr(changed, 1u);
}
}  // namespace

cudaError_t forest_roots_weighted(Runtime& rt, uint32_t n, const uint32_t* parent, const double* wv,
                                  uint32_t* root, double* prod) {
  if (n == 0) return cudaSuccess;
  cudaStream_t st = rt.st;
  uint32_t* tmp = rt.alloc<uint32_t>(n);
  double* ptmp = rt.alloc<double>(n);
  uint32_t* ctr = rt.alloc<uint32_t>(1);
  if (rt.err) return rt.err;
  k_root_init_w<<<grid_for(n), 256, 0, st>>>(n, parent, wv, root, prod);
  ++rt.launches;
  uint32_t* a = root;
  uint32_t* b = tmp;
  double* pa = prod;
  double* pb = ptmp;
  int rounds = 0;
  for (int batch = 8;; batch = 4) {
    cudaMemsetAsync(ctr, 0, sizeof(uint32_t), st);
    for (int j = 0; j < batch; ++j) {
      k_root_jump_w<<<grid_for(n), 256, 0, st>>>(n, a, pa, b, pb, ctr);
      std::swap(a, b);
      std::swap(pa, pb);
    }
    rt.launches += batch;
    rounds += batch;
    rt.read(ctr, 1);
    if (!rt.h_cnt[0] || rt.err) break;
    if (rounds > kMaxJump) {
      k_set_flag<<<1, 1, 0, st>>>(rt.d_status, ST_CYCLE);
      ++rt.launches;
      break;
    }
  }
  if (a != root) {
    cudaMemcpyAsync(root, a, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(prod, pa, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
  }
  rt.free(tmp);
  rt.free(ptmp);
  rt.free(ctr);
  return rt.err ? rt.err : cudaGetLastError();
}

}  // namespace fa
