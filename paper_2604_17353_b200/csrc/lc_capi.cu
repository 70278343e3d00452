// ABI-level helpers: version, status strings, thread-local last error.
#include <stdio.h>
#include <string.h>

#include "lc_common.cuh"

static thread_local char g_last_error[512] = "";

void lcb_set_last_error(const char* msg, const char* file, int line) {
  snprintf(g_last_error, sizeof(g_last_error), "%s (%s:%d)", msg, file, line);
}

extern "C" int lc_abi_version(void) { return LC_ABI_VERSION; }

extern "C" const char* lc_last_error(void) { return g_last_error; }

extern "C" const char* lc_status_string(int status) {
  switch (status) {
    case LC_OK: return "ok";
    case LC_E_CONFIG: return "config error";
    case LC_E_ZERO_MASS: return "no probability mass";
    case LC_E_CAPACITY: return "capacity exhausted";
    case LC_E_CUDA: return "CUDA error";
    case LC_E_ARG: return "bad argument";
    case LC_E_STATE: return "write-back prefix no longer live";
    default: return "unknown status";
  }
}
