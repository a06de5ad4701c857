// Run-time binding of NCCL (see hzg_nccl.h).
#include <dlfcn.h>

#include <cstdlib>
#include <mutex>

#include "hzg_nccl.h"

namespace hzg {
namespace nccl {

namespace {

Api g_api{};
bool g_loaded = false;
std::string g_err;
std::once_flag g_once;

template <class F>
bool sym(void* h, const char* name, F& out) {
  out = reinterpret_cast<F>(dlsym(h, name));
  if (!out) g_err = std::string("NCCL symbol missing: ") + name;
  return out != nullptr;
}

void do_load() {
  void* h = nullptr;
  if (const char* path = std::getenv("HZG_NCCL_LIB")) {
    h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
  } else {
    // the process's NCCL (PyTorch loads libnccl.so.2 with libtorch_cuda)
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  }
  if (!h) {
    g_err = std::string("cannot load NCCL: ") + dlerror();
    return;
  }
  bool ok = sym(h, "ncclGetUniqueId", g_api.GetUniqueId) && sym(h, "ncclCommInitRank", g_api.CommInitRank) &&
            sym(h, "ncclCommInitAll", g_api.CommInitAll) &&
            sym(h, "ncclCommDestroy", g_api.CommDestroy) &&
            sym(h, "ncclCommGetAsyncError", g_api.CommGetAsyncError) &&
            sym(h, "ncclGroupStart", g_api.GroupStart) && sym(h, "ncclGroupEnd", g_api.GroupEnd) &&
            sym(h, "ncclSend", g_api.Send) && sym(h, "ncclRecv", g_api.Recv) &&
            sym(h, "ncclAllReduce", g_api.AllReduce) && sym(h, "ncclGetErrorString", g_api.GetErrorString) &&
            sym(h, "ncclGetVersion", g_api.GetVersion);
  g_loaded = ok;
}

}  // namespace

const Api* load(std::string& err) {
  std::call_once(g_once, do_load);
  if (!g_loaded) {
    err = g_err;
    return nullptr;
  }
  return &g_api;
}

}  // namespace nccl
}  // namespace hzg
