// api.cu -- error plumbing and version of libfct.so
#include <string.h>
#include <atomic>
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

static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
uint64_t launches() { return g_launches.load(std::memory_order_relaxed); }

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
extern "C" uint64_t fct_launch_count(void) { return fct::launches(); }
