// hshard-b200: run-time NCCL binding (see nccl_dyn.hpp).
#include "nccl_dyn.hpp"

#include <dlfcn.h>

#include <mutex>
#include <string>

#include "hshard/common.hpp"

namespace hshard::exec::nccl {

namespace {

template <class F>
void bind(void* lib, F& fn, const char* name) {
  fn = reinterpret_cast<F>(dlsym(lib, name));
  if (!fn) fail(Errc::CommError, std::string("NCCL symbol missing: ") + name);
}

}  // namespace

const Api& api() {
  static Api a{};
  static std::once_flag once;
  static std::string error;
  std::call_once(once, [] {
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's, if loaded
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!lib) {
      error = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    try {
      bind(lib, a.GetUniqueId, "ncclGetUniqueId");
      bind(lib, a.CommInitRank, "ncclCommInitRank");
      bind(lib, a.CommDestroy, "ncclCommDestroy");
      bind(lib, a.GetErrorString, "ncclGetErrorString");
      bind(lib, a.GroupStart, "ncclGroupStart");
      bind(lib, a.GroupEnd, "ncclGroupEnd");
      bind(lib, a.Send, "ncclSend");
      bind(lib, a.Recv, "ncclRecv");
    } catch (const Error& e) {
      error = e.what();
    }
  });
  if (!error.empty()) fail(Errc::CommError, error);
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(Errc::CommError, std::string(what) + ": " + api().GetErrorString(r));
}

}  // namespace hshard::exec::nccl
