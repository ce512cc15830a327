// abi.cu -- error reporting and version of the C ABI (include/ss_abi.h).
#include <string.h>
#include "ss_common.cuh"

namespace {
thread_local char g_err[256] = "";
}

void ss_set_error(const char *msg) {
    strncpy(g_err, msg ? msg : "", sizeof(g_err) - 1);
    g_err[sizeof(g_err) - 1] = 0;
}

extern "C" const char *ss_last_error(void) { return g_err; }
extern "C" int ss_version(void) { return 1; }
