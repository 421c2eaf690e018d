// paper_1711_04471_b200/csrc/sw2d_nccl.cuh — NCCL loaded at run time.
//
// Single-GPU handles never touch NCCL; multi-rank handles dlopen
// libnccl.so.2 (the CUDA image's NCCL 2.28, the same library torch uses) on
// first use, so the library has no link-time NCCL dependency.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

namespace sw2d_host {

struct NcclApi {
  bool ok = false;
  const char* why = "not loaded";
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t,
                            ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// Loads once (thread-safe); returns the table (check .ok).
const NcclApi& nccl();

// CUDA driver stream memory operations (P2P halo signalling), resolved with
// cudaGetDriverEntryPoint.  Values are 32-bit; wait is ">=".
struct MemOps {
  bool ok = false;
  int (*write32)(cudaStream_t, unsigned long long addr, unsigned value, unsigned flags) = nullptr;
  int (*wait32)(cudaStream_t, unsigned long long addr, unsigned value, unsigned flags) = nullptr;
};
const MemOps& memops();

}  // namespace sw2d_host
