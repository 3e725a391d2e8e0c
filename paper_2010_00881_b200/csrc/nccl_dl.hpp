// nccl_dl.hpp -- NCCL loaded at run time (dlopen): the library has no link-time NCCL
// dependency, so the CPU tests can load it, and on a GPU box it binds to the libnccl.so.2
// that PyTorch already loaded into the process (one NCCL per process).
#pragma once
#include <dlfcn.h>
#include <nccl.h>

namespace fcm {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

inline NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return a;
#define FCM_SYM(name) a.name = reinterpret_cast<decltype(a.name)>(dlsym(lib, "nccl" #name))
    FCM_SYM(GetUniqueId);
    FCM_SYM(CommInitRank);
    FCM_SYM(CommDestroy);
    FCM_SYM(GroupStart);
    FCM_SYM(GroupEnd);
    FCM_SYM(Send);
    FCM_SYM(Recv);
    FCM_SYM(AllReduce);
    FCM_SYM(AllGather);
    FCM_SYM(GetErrorString);
#undef FCM_SYM
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.GroupStart && a.GroupEnd && a.Send &&
           a.Recv && a.AllReduce && a.AllGather && a.GetErrorString;
    return a;
  }();
  return api;
}

}  // namespace fcm
