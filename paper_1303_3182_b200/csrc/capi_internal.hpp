// Internal definitions shared by the C-ABI translation units.
#pragma once
#include <string>
#include <vector>

#include "../../include/tqr.h"
#include "sched.hpp"

struct tqr_build {
  tqr::Build* b = nullptr;
  std::vector<tqr::Edge> edges;
  bool have_edges = false;
  ~tqr_build() { delete b; }
};

namespace tqr {
// thread-local last error (tqr_last_error)
extern thread_local std::string g_err;

// Run f, mapping C++ exceptions onto TQR_E* status codes + tqr_last_error().
template <class F>
inline int guard(F&& f) {
  try {
    f();
    return TQR_OK;
  } catch (const ValueError& e) {
    g_err = e.what();
    return TQR_EVALUE;
  } catch (const KeyError& e) {
    g_err = e.what();
    return TQR_EKEY;
  } catch (const AssertError& e) {
    g_err = e.what();
    return TQR_EASSERT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return TQR_EOTHER;
  }
}

}  // namespace tqr
