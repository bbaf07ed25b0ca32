// dist.cu -- multi-GPU entry points (H7).  NCCL is loaded at run time
// (dlopen of the torch-bundled libnccl.so.2) so libfa has no link-time NCCL
// dependency and one process never holds two NCCL copies.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <string>

#include "fa.h"

extern "C" {

fa_status fa_nccl_unique_id(void* out128) {
  if (!out128) return FA_E_ARG;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return FA_E_NCCL;
  typedef int (*get_id_t)(void*);
  get_id_t fn = (get_id_t)dlsym(h, "ncclGetUniqueId");
  if (!fn) return FA_E_NCCL;
  return fn(out128) == 0 ? FA_OK : FA_E_NCCL;
}

fa_status fa_accumulate_dist(fa_ctx* ctx, const void* nccl_id128, int rank, int nranks,
                             int64_t global_rows, int64_t cols, int64_t row_begin, int64_t local_rows,
                             const float* dem, float nodata, const uint8_t* dirs, const void* w,
                             fa_wtype wtype, void* acc, fa_atype atype) {
  (void)ctx; (void)nccl_id128; (void)rank; (void)nranks; (void)global_rows; (void)cols;
  (void)row_begin; (void)local_rows; (void)dem; (void)nodata; (void)dirs; (void)w; (void)wtype;
  (void)acc; (void)atype;
  return FA_E_STATE;
}

}  // extern "C"
