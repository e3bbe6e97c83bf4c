#include "cpsel_nccl.h"

#include <dlfcn.h>

#include <mutex>

namespace cpsel {

static NcclApi g_api;
static std::once_flag g_once;

template <typename F> static bool sym(void* h, const char* name, F& out) {
  out = reinterpret_cast<F>(dlsym(h, name));
  return out != nullptr;
}

static void load() {
  // Prefer an NCCL already mapped into the process (torch's), then the system one.
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    g_api.load_error = "libnccl.so.2 not found (dlopen failed)";
    return;
  }
  bool ok = sym(h, "ncclGetUniqueId", g_api.GetUniqueId) && sym(h, "ncclCommInitRank", g_api.CommInitRank) &&
            sym(h, "ncclCommDestroy", g_api.CommDestroy) && sym(h, "ncclAllGather", g_api.AllGather) &&
            sym(h, "ncclBroadcast", g_api.Broadcast) && sym(h, "ncclAllReduce", g_api.AllReduce) &&
            sym(h, "ncclGroupStart", g_api.GroupStart) && sym(h, "ncclGroupEnd", g_api.GroupEnd) &&
            sym(h, "ncclGetErrorString", g_api.GetErrorString);
  if (!ok) {
    g_api.load_error = "libnccl.so.2 lacks a required symbol";
    return;
  }
  sym(h, "ncclCommGetAsyncError", g_api.CommGetAsyncError);
  sym(h, "ncclCommAbort", g_api.CommAbort);
  g_api.ok = true;
}

const NcclApi& nccl_api() {
  std::call_once(g_once, load);
  return g_api;
}

}  // namespace cpsel
