// tacos_nccl.cpp -- run-time binding of NCCL (see tacos_nccl.h).
#include "tacos_nccl.h"

#include <dlfcn.h>
#include <link.h>

#include <cstdlib>
#include <mutex>

namespace tacos {
namespace {
std::once_flag g_once;
NcclApi g_api;
bool g_ok = false;
std::string g_err;

template <typename F>
bool sym(void *h, const char *name, F *out) {
  *out = reinterpret_cast<F>(dlsym(h, name));
  if (!*out) g_err = std::string("NCCL symbol ") + name + " missing";
  return *out != nullptr;
}

void load() {
  void *h = nullptr;
  const char *env = getenv("TACOS_NCCL_LIB");
  if (env && *env) {
    h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  } else {
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process (PyTorch's)
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  }
  if (!h) {
    const char *e = dlerror();
    g_err = std::string("cannot load NCCL: ") + (e ? e : "not found");
    return;
  }
  bool ok = sym(h, "ncclGetVersion", &g_api.GetVersion) && sym(h, "ncclGetUniqueId", &g_api.GetUniqueId) &&
            sym(h, "ncclCommInitRank", &g_api.CommInitRank) && sym(h, "ncclCommInitAll", &g_api.CommInitAll) &&
            sym(h, "ncclCommDestroy", &g_api.CommDestroy) && sym(h, "ncclAllReduce", &g_api.AllReduce) &&
            sym(h, "ncclGetErrorString", &g_api.GetErrorString);
  if (!ok) return;
  struct link_map *lm = nullptr;
  if (dlinfo(h, RTLD_DI_LINKMAP, &lm) == 0 && lm && lm->l_name) g_api.path = lm->l_name;
  g_ok = true;
}
}  // namespace

const NcclApi *nccl_api(std::string *err) {
  std::call_once(g_once, load);
  if (!g_ok && err) *err = g_err;
  return g_ok ? &g_api : nullptr;
}
}  // namespace tacos
