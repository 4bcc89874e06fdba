// hshard-b200 C ABI internals: opaque handle layouts and error translation.
#pragma once

#include <memory>
#include <new>
#include <optional>
#include <string>

#include "hshard/resolve.hpp"
#include "hshard/switch.hpp"
#include "hshard_c.h"

struct hs_plan {
  std::optional<hshard::CommPlan> comm;
  std::optional<hshard::SwitchPlan> sw;
};

namespace hshard::capi {

extern thread_local std::string g_last_error;
int fail_code(Errc e, const std::string& msg);
char* dup_string(const std::string& s);
Shape to_shape(const int64_t* shape, int ndim);
DType to_dtype(int code);

// Runs fn, translating exceptions into 1 + Errc (never throws across the ABI).
template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const Error& e) {
    return fail_code(e.code(), e.what());
  } catch (const std::bad_alloc& e) {
    return fail_code(Errc::CudaError, std::string("out of memory: ") + e.what());
  } catch (const std::exception& e) {
    return fail_code(Errc::ParseError, e.what());
  }
}

}  // namespace hshard::capi
