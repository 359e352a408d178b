// NCCL access for the block-sharded multi-GPU path, resolved at run time.
//
// libnccl.so.2 is dlopen'ed (in a torch process this returns the NCCL torch
// already loaded, so one NCCL instance serves both), keeping the library
// loadable on hosts without NCCL for the single-GPU path.
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include "nccl_shim.h"
#include "status.h"

namespace cb {

NcclApi& nccl_api() {
  static NcclApi api;
  return api;
}

int nccl_load() {
  NcclApi& a = nccl_api();
  if (a.loaded) return CB_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    set_error("NCCL not available: %s", dlerror());
    return CB_ERR_UNSUPPORTED;
  }
#define SYM(name) a.name = (decltype(a.name))dlsym(h, #name)
  SYM(ncclGetUniqueId);
  SYM(ncclCommInitRank);
  SYM(ncclCommDestroy);
  SYM(ncclAllGather);
  SYM(ncclAllReduce);
  SYM(ncclGroupStart);
  SYM(ncclGroupEnd);
  SYM(ncclGetErrorString);
#undef SYM
  if (!a.ncclGetUniqueId || !a.ncclCommInitRank || !a.ncclAllGather || !a.ncclAllReduce) {
    set_error("NCCL symbols missing");
    return CB_ERR_UNSUPPORTED;
  }
  a.loaded = true;
  return CB_OK;
}

int nccl_fail(int r, const char* what) {
  NcclApi& a = nccl_api();
  set_error("NCCL error %d (%s) in %s", r,
            a.ncclGetErrorString ? a.ncclGetErrorString((ncclResult_t)r) : "?", what);
  return CB_ERR_CUDA;
}

}  // namespace cb

using namespace cb;

extern "C" {

int cb_nccl_unique_id(void* out128) {
  int rc = nccl_load();
  if (rc) return rc;
  ncclUniqueId id;
  ncclResult_t r = nccl_api().ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(out128, &id, sizeof(id));
  return CB_OK;
}

int cb_nccl_comm_init(const void* unique_id128, int world_size, int rank, void** comm) {
  int rc = nccl_load();
  if (rc) return rc;
  ncclUniqueId id;
  memcpy(&id, unique_id128, sizeof(id));
  ncclComm_t c;
  ncclResult_t r = nccl_api().ncclCommInitRank(&c, world_size, id, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  *comm = (void*)c;
  return CB_OK;
}

int cb_nccl_comm_destroy(void* comm) {
  if (!comm) return CB_OK;
  int rc = nccl_load();
  if (rc) return rc;
  ncclResult_t r = nccl_api().ncclCommDestroy((ncclComm_t)comm);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
  return CB_OK;
}

}  // extern "C"
