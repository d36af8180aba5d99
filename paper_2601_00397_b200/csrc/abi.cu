// abi.cu — error reporting and bookkeeping shared by every libtwb200 entry point.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace twb {

static thread_local char g_err[512] = "";
static thread_local int64_t g_launches = 0;

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return TW_ECUDA;
  }
  return TW_OK;
}

void count_launch() { ++g_launches; }

}  // namespace twb

extern "C" {

int tw_abi_version(void) { return TWB200_ABI_VERSION; }
const char* tw_last_error(void) { return twb::g_err; }
int64_t tw_launch_count(void) { return twb::g_launches; }

}  // extern "C"
