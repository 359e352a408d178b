// Run-time resolved NCCL entry points (see nccl_shim.cu).
#pragma once
#include <nccl.h>

namespace cb {

struct NcclApi {
  bool loaded = false;
  ncclResult_t (*ncclGetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*ncclCommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*ncclCommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*ncclAllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  ncclResult_t (*ncclAllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*ncclGroupStart)() = nullptr;
  ncclResult_t (*ncclGroupEnd)() = nullptr;
  const char* (*ncclGetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api();
int nccl_load();
int nccl_fail(int r, const char* what);

}  // namespace cb
