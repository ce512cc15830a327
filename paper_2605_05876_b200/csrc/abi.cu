// abi.cu -- error reporting, version and per-device launch helpers of the C
// ABI (include/ss_abi.h).
#include <string.h>
#include <map>
#include <mutex>
#include <utility>
#include "ss_common.cuh"

namespace {
thread_local char g_err[256] = "";
constexpr int kMaxDevices = 64;
int g_sms[kMaxDevices] = {0};
std::mutex g_attr_mu;
std::map<std::pair<int, const void *>, int> g_attr_max;  // (device, kernel) -> opt-in set so far

int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}
}  // namespace

void ss_set_error(const char *msg) {
    strncpy(g_err, msg ? msg : "", sizeof(g_err) - 1);
    g_err[sizeof(g_err) - 1] = 0;
}

int ss_sm_count() {
    const int dev = current_device();
    if (dev < 0 || dev >= kMaxDevices) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v > 0 ? v : 148;
    }
    int v = __atomic_load_n(&g_sms[dev], __ATOMIC_RELAXED);
    if (v == 0) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (v <= 0) v = 148;
        __atomic_store_n(&g_sms[dev], v, __ATOMIC_RELAXED);
    }
    return v;
}

void ss_func_smem(const void *func, int bytes) {
    // the attribute is an upper bound: only ever raise it, so a launch with
    // less dynamic shared memory than an earlier one never needs a call
    const auto key = std::make_pair(current_device(), func);
    std::lock_guard<std::mutex> lock(g_attr_mu);
    auto it = g_attr_max.find(key);
    if (it != g_attr_max.end() && it->second >= bytes) return;
    if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess)
        g_attr_max[key] = bytes;
}

extern "C" const char *ss_last_error(void) { return g_err; }
extern "C" int ss_version(void) { return 2; }
