// Test-infrastructure shim over the reference (femopt) — NOT product code.
//
// libfemopt's C API (proj/include/femopt.h:44-76) exposes parse / optimize /
// emit_c / flops / verify but not the tree-walking interpreter that the
// reference itself uses as its oracle (proj/src/interp.cpp:125-154,
// `interpret`).  This file adds exactly that one entry point so the golden
// fixtures under tests/golden/ can be produced by the reference's own
// executor.  Compiled together with the reference sources in place by
// oracle/Makefile; output goes to oracle/_ref/ only.
#include <cstring>
#include <string>

#include "interp.hpp"
#include "json_io.hpp"

namespace {
thread_local std::string g_err;
}

extern "C" {

// Interprets the kernel given as IR JSON text and copies output `name`
// (row-major, as interp.cpp stores it) into out[0..n).  Returns the number of
// values the output has, or -1 on failure (message via refshim_last_error).
long refshim_interpret(const char* json_text, const char* name, double* out, long n) {
  try {
    femopt::Kernel k = femopt::kernel_from_json(json_text);
    auto res = femopt::interpret(k);
    auto it = res.find(name);
    if (it == res.end()) {
      g_err = std::string("no output named ") + name;
      return -1;
    }
    long m = static_cast<long>(it->second.size());
    if (out) std::memcpy(out, it->second.data(), sizeof(double) * static_cast<size_t>(m < n ? m : n));
    return m;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

const char* refshim_last_error(void) { return g_err.c_str(); }

}  // extern "C"
