// Error reporting and version of the C ABI (include/idsketch_b200.h).
#include <stdio.h>
#include <string.h>

#include <atomic>

#include "common.cuh"

static thread_local char g_last_error[512] = "";

void ids_set_last_error(const char* msg) {
    strncpy(g_last_error, msg ? msg : "", sizeof(g_last_error) - 1);
    g_last_error[sizeof(g_last_error) - 1] = '\0';
}

void ids_set_cuda_error(cudaError_t e, const char* file, int line) {
    const char* base = strrchr(file, '/');
    snprintf(g_last_error, sizeof(g_last_error), "%s (%s:%d)", cudaGetErrorString(e),
             base ? base + 1 : file, line);
}

extern "C" const char* ids_last_error(void) { return g_last_error; }

extern "C" int ids_version(void) { return 1; }

static std::atomic<long long> g_launches{0};

void ids_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

extern "C" int64_t ids_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int ids_sm_count() {
    static int sms = [] {
        int dev = 0, n = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) {
            cudaGetLastError();
            return 148;  // B200
        }
        return n;
    }();
    return sms;
}
