// nccl_shim.h -- NCCL entry points resolved at run time (dlopen), so the
// library has no link-time NCCL dependency: single-GPU use never loads NCCL,
// and a process that already loaded one (e.g. torch's bundled libnccl.so.2)
// shares it instead of clashing with a second copy.
#pragma once

#include <nccl.h>

namespace ab2 {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};

// Throws ab2::Error(ALSNCG_ENCCL) if no libnccl.so.2 can be loaded.
const NcclApi& nccl();

}  // namespace ab2
