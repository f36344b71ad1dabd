// NCCL entry points resolved at run time (dlopen of libnccl.so.2, the copy
// the PyTorch process has already loaded), so that the library links and
// loads on machines without NCCL and single-GPU use never touches it.
#pragma once
#include <cuda_runtime.h>

#include <string>

namespace hmg {

typedef struct ncclComm* ncclComm_t;
struct NcclUniqueId {
    char internal[128];
};
enum { kNcclSuccess = 0, kNcclFloat64 = 8, kNcclSum = 0 };

struct Nccl {
    int (*GetUniqueId)(NcclUniqueId*) = nullptr;
    int (*CommInitRank)(ncclComm_t*, int, NcclUniqueId, int) = nullptr;
    int (*CommDestroy)(ncclComm_t) = nullptr;
    int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
};

// Loaded table, or nullptr with `err` set.  HMG_TRANSPORT=local selects the
// TEST-ONLY in-process transport (local_transport.cu, built separately into
// libhmg_localtx.so and loaded from next to this library: all ranks threads
// of one process on one GPU, for testing the multi-GPU path on one device).
const Nccl* nccl(std::string* err);

}  // namespace hmg
