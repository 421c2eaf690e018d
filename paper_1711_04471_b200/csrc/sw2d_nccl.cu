// paper_1711_04471_b200/csrc/sw2d_nccl.cu — run-time NCCL loader.
#include "sw2d_nccl.cuh"

#include <dlfcn.h>

#include <cstdlib>
#include <mutex>
#include <string>

namespace sw2d_host {

namespace {

NcclApi g_api;
std::once_flag g_once;

void* open_nccl() {
  const char* env = std::getenv("SW2D_NCCL_LIBRARY");
  if (env && *env) {
    if (void* h = dlopen(env, RTLD_NOW | RTLD_GLOBAL)) return h;
  }
  if (void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL)) return h;
  // the CUDA image's NCCL (the one torch loads), relative to this library
  Dl_info info;
  if (dladdr(reinterpret_cast<void*>(&open_nccl), &info) && info.dli_fname) {
    std::string self(info.dli_fname);
    const std::string key = "/site-packages/";
    const size_t p = self.find(key);
    if (p != std::string::npos) {
      std::string path = self.substr(0, p + key.size()) + "nvidia/nccl/lib/libnccl.so.2";
      if (void* h = dlopen(path.c_str(), RTLD_NOW | RTLD_GLOBAL)) return h;
    }
  }
  const char* fallback =
      "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2";
  return dlopen(fallback, RTLD_NOW | RTLD_GLOBAL);
}

template <typename F>
bool sym(void* h, const char* name, F& out) {
  out = reinterpret_cast<F>(dlsym(h, name));
  return out != nullptr;
}

void load() {
  void* h = open_nccl();
  if (!h) {
    g_api.why = "cannot dlopen libnccl.so.2";
    return;
  }
  bool ok = sym(h, "ncclGetUniqueId", g_api.GetUniqueId) &&
            sym(h, "ncclCommInitRank", g_api.CommInitRank) &&
            sym(h, "ncclCommDestroy", g_api.CommDestroy) &&
            sym(h, "ncclCommGetAsyncError", g_api.CommGetAsyncError) &&
            sym(h, "ncclSend", g_api.Send) && sym(h, "ncclRecv", g_api.Recv) &&
            sym(h, "ncclAllReduce", g_api.AllReduce) &&
            sym(h, "ncclAllGather", g_api.AllGather) &&
            sym(h, "ncclGroupStart", g_api.GroupStart) &&
            sym(h, "ncclGroupEnd", g_api.GroupEnd) &&
            sym(h, "ncclGetErrorString", g_api.GetErrorString);
  if (!ok) {
    g_api.why = "libnccl.so.2 lacks a required symbol";
    return;
  }
  g_api.ok = true;
  g_api.why = "";
}

}  // namespace

const NcclApi& nccl() {
  std::call_once(g_once, load);
  return g_api;
}

namespace {
MemOps g_memops;
std::once_flag g_memops_once;

void load_memops() {
  void* w = nullptr;
  void* v = nullptr;
  cudaDriverEntryPointQueryResult q1, q2;
  if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &q1) != cudaSuccess ||
      cudaGetDriverEntryPoint("cuStreamWaitValue32", &v, cudaEnableDefault, &q2) != cudaSuccess ||
      q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || !w || !v)
    return;
  g_memops.write32 = reinterpret_cast<decltype(g_memops.write32)>(w);
  g_memops.wait32 = reinterpret_cast<decltype(g_memops.wait32)>(v);
  g_memops.ok = true;
}
}  // namespace

const MemOps& memops() {
  std::call_once(g_memops_once, load_memops);
  return g_memops;
}

}  // namespace sw2d_host
