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

// last kernel instance launched per hot-path stage ("sketch", "rownorm"), for evidence matching (bench.py)
static char g_inst[2][128];
static std::atomic<int> g_inst_lock{0};
void set_instance(int slot, const char* fmt, ...) {
  char buf[128];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  while (g_inst_lock.exchange(1)) {}
  memcpy(g_inst[slot], buf, sizeof(buf));
  g_inst_lock.store(0);
}
int get_instance(int slot, char* out, size_t len) {
  if (!out || len == 0 || slot < 0 || slot > 1) return -1;
  while (g_inst_lock.exchange(1)) {}
  snprintf(out, len, "%s", g_inst[slot]);
  g_inst_lock.store(0);
  return 0;
}

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
extern "C" int fct_last_instance(int32_t stage, char* buf, size_t len) { return fct::get_instance(stage, buf, len); }
