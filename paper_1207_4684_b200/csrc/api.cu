// api.cu -- error plumbing and version of libfct.so
#include <string.h>
#include "common.cuh"

namespace fct {
static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
const char* get_error() { return g_err; }

bool debug_sync() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FCT_DEBUG");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}
}  // namespace fct

extern "C" const char* fct_last_error(void) { return fct::get_error(); }
extern "C" const char* fct_version(void) { return "fct-b200 0.1 sm_100a"; }
