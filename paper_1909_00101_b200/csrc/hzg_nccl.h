// NCCL entry points used by libhzg's multi-GPU data plane, resolved at run
// time (dlopen) so that the library binds to the NCCL build the host
// process already loaded (PyTorch's, when the caller is a torch process)
// instead of carrying its own copy: two NCCL builds in one process would
// not share communicators, proxies or their CUDA-graph support.
#pragma once
#include <nccl.h>

#include <string>

namespace hzg {
namespace nccl {

struct Api {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
  ncclResult_t (*GetVersion)(int*);
};

// Resolve the entry points once (HZG_NCCL_LIB names an explicit library;
// otherwise an already loaded libnccl.so.2, then the loader's search path).
// Returns nullptr and sets `err` when NCCL is unavailable.
const Api* load(std::string& err);

}  // namespace nccl
}  // namespace hzg
