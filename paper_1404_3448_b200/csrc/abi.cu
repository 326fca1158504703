// abi.cu -- error reporting and version entry points of libsaix_b200.so.
#include <cstdarg>

#include "common.cuh"

namespace saix {

static thread_local char g_last_error[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
    va_end(ap);
}

}  // namespace saix

extern "C" const char *saix_last_error(void) { return saix::g_last_error; }

extern "C" int saix_abi_version(void) { return 1; }
