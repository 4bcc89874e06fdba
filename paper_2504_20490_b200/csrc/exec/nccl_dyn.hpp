// hshard-b200: NCCL entry points resolved at run time.
//
// libhshard_b200.so never links libnccl: a process that loads it before
// torch would otherwise bind libnccl.so.2 to the system NCCL and break
// torch's own (newer) NCCL symbols.  Only the HS_PROG_NCCL baseline needs
// NCCL; its first use dlopen()s "libnccl.so.2" -- reusing the copy torch
// already loaded when there is one.
#pragma once

#include <nccl.h>

namespace hshard::exec::nccl {

struct Api {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  const char* (*GetErrorString)(ncclResult_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
};

// Loads the library on first call; throws Errc::CommError if unavailable.
const Api& api();
// Throws Errc::CommError with NCCL's message when r != ncclSuccess.
void check(ncclResult_t r, const char* what);

}  // namespace hshard::exec::nccl
