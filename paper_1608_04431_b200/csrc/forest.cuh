// forest.cuh -- device forest accumulation: S(v) = val(v) + sum_{children c} S(c)
// for a forest given by explicit parent pointers.  Used for the block-exit
// graph G1 and the tile perimeter graph G2 ("solved using the same
// strategy described in Algorithm 1").
#pragma once
#include "fa_internal.cuh"

namespace fa {

struct Runtime {
  cudaStream_t st = nullptr;
  uint32_t* d_cnt = nullptr;     // device scratch counters [16]
  uint32_t* h_cnt = nullptr;     // pinned host mirror [16]
  uint32_t* d_status = nullptr;  // status word (ST_*)
  // statistics
  int64_t peel_rounds = 0, contract_levels = 0, jump_rounds = 0, launches = 0;
  int walk_cap = 128;  // steps per graph walk before re-queueing (FA_OPT_WALK_CAP; 0 = peel only)
  bool device_solver = false;  // FA_OPT_GRAPH: forest_dev.cu (one cooperative launch per solve)
  bool use_device_solver(uint32_t) const { return device_solver; }
  cudaError_t err = cudaSuccess;

  template <class U>
  U* alloc(size_t n) {
    void* p = nullptr;
    if (n == 0) n = 1;
    cudaError_t e = cudaMallocAsync(&p, n * sizeof(U), st);
    if (e != cudaSuccess && err == cudaSuccess) err = e;
    return static_cast<U*>(p);
  }
  void free(void* p) {
    if (p) cudaFreeAsync(p, st);
  }
  // read n device counters into h_cnt (synchronises the stream)
  cudaError_t read(const uint32_t* d, int n) {
    cudaError_t e = cudaMemcpyAsync(h_cnt, d, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess && err == cudaSuccess) err = e;
    return e;
  }
};

template <class T>
cudaError_t forest_solve(Runtime& rt, uint32_t n, const uint32_t* parent, T* val);
// the same solve as one cooperative persistent kernel (forest_dev.cu); done =
// false when it could not run (no cooperative launch, scratch pool too small)
template <class T>
cudaError_t forest_solve_device(Runtime& rt, uint32_t n, const uint32_t* parent, T* val, bool& done);
cudaError_t forest_solve_weighted_device(Runtime& rt, uint32_t n, const uint32_t* parent, const double* wv,
                                         double* val, bool& done);
// the same without a host read: node count *n_dev (<= n_max), statistics to
// stats_out[0..2] (device), scratch overflow -> ST_RETRY in the status word;
// cudaErrorNotSupported when a cooperative launch is not possible
template <class T>
cudaError_t forest_solve_device_async(Runtime& rt, uint32_t n_max, const uint32_t* n_dev, const uint32_t* parent,
                                      T* val, uint32_t* stats_out);
// absorption: S(v) = val(v) + sum_children wv(c) S(c)
cudaError_t forest_solve_weighted(Runtime& rt, uint32_t n, const uint32_t* parent, const double* wv, double* val);
// absorption: roots plus the product of edge weights from each node up to its root
cudaError_t forest_roots_weighted(Runtime& rt, uint32_t n, const uint32_t* parent, const double* wv,
                                  uint32_t* root, double* prod);

// root of every node in a forest (pointer jumping); cycles -> ST_CYCLE
cudaError_t forest_roots(Runtime& rt, uint32_t n, const uint32_t* parent, uint32_t* root);
// the same as one cooperative launch (forest_dev.cu); cudaErrorNotSupported when that is not possible
cudaError_t forest_roots_device(Runtime& rt, uint32_t n, const uint32_t* parent, uint32_t* root);

inline unsigned grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 64) g = 148 * 64;  // grid-stride beyond this
  return (unsigned)g;
}

}  // namespace fa
