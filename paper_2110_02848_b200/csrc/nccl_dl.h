// nccl_dl.h -- NCCL entry points resolved at run time (dlopen "libnccl.so.2"): libfstc builds without
// NCCL and uses the copy the process already has (PyTorch's bundled NCCL) when the sharded mode runs.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace fstc {

typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
enum { kNcclUint32 = 3, kNcclUint64 = 5 };  // ncclDataType_t
enum { kNcclSum = 0 };                      // ncclRedOp_t

struct NcclApi {
  bool ok = false;
  int (*GetUniqueId)(ncclUniqueId*) = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};

// Loads the API once; returns nullptr (and sets the library error) if NCCL is unavailable.
const NcclApi* nccl_api();

}  // namespace fstc

struct fst_comm {
  fstc::ncclComm_t comm = nullptr;
  int world = 1;
  int rank = 0;
};
