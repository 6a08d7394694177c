// Library-wide state of the C-ABI (include/iedd_b200.h): error text and the
// launch counter reported as bench.py's gpu_launches.
#include <string>

#include "common.cuh"

struct ie_matvec;

namespace ie {
std::atomic<int64_t> g_launches{0};
static thread_local std::string t_err;
void set_error(const std::string& msg) { t_err = msg; }
}  // namespace ie

extern "C" const char* ie_last_error(void) { return ie::t_err.c_str(); }
extern "C" int64_t ie_launch_count(void) { return ie::g_launches.load(); }
