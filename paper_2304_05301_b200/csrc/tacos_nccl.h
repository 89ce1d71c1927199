// tacos_nccl.h -- NCCL, resolved at run time (product side; used only by the cross-GPU
// best-of-S selection: one 16-byte ncclAllReduce MIN of the two best keys).
//
// libtacos.so does not link NCCL: the first multi-GPU call dlopen()s it, preferring a
// libnccl.so.2 already mapped into the process (e.g. the one PyTorch loaded), so the
// library loads on hosts without NCCL and never pins a second NCCL next to the caller's.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <string>

namespace tacos {
struct NcclApi {
  ncclResult_t (*GetVersion)(int *);
  ncclResult_t (*GetUniqueId)(ncclUniqueId *);
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
  ncclResult_t (*CommInitAll)(ncclComm_t *, int, const int *);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  const char *(*GetErrorString)(ncclResult_t);
  std::string path;  // the shared object the symbols come from
};
// The loaded API, or nullptr with *err set (TACOS_NCCL_LIB names a library to use instead).
const NcclApi *nccl_api(std::string *err);
}  // namespace tacos
