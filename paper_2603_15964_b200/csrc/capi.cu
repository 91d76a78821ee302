// capi.cu -- library-level entry points of liblmep (status strings, errors).
#include <stdio.h>
#include <string.h>

#include "common.cuh"

namespace lmep {

static thread_local char g_last_error[512] = "";
static std::atomic<int64_t> g_launches{0};

void set_last_error(const char *what, cudaError_t e)
{
    snprintf(g_last_error, sizeof(g_last_error), "%s: %s", what, cudaGetErrorString(e));
}

void set_last_error_text(const char *what, const char *msg)
{
    snprintf(g_last_error, sizeof(g_last_error), "%s: %s", what, msg);
}

void count_launches(int64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

int current_device()
{
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) dev = 0;
    return dev < kMaxDevices ? dev : kMaxDevices - 1;
}

static std::atomic<int> g_sms[kMaxDevices];

int device_sm_count()
{
    const int dev = current_device();
    int v = g_sms[dev].load(std::memory_order_relaxed);
    if (v <= 0) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
            v = 148;
        g_sms[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

static DeviceSettings g_settings[kMaxDevices];

DeviceSettings &device_settings() { return g_settings[current_device()]; }

int launch_status(const char *what)
{
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_last_error(what, e);
        return LMEP_CUDA_ERROR;
    }
    return LMEP_OK;
}

}  // namespace lmep

extern "C" int lmep_version(void) { return 100; }

extern "C" const char *lmep_status_string(int status)
{
    switch (status) {
    case LMEP_OK: return "ok";
    case LMEP_NONFINITE: return "non-finite value";
    case LMEP_DIMENSION: return "dimension mismatch";
    case LMEP_INVALID_CONFIG: return "invalid configuration";
    case LMEP_CUDA_ERROR: return "CUDA error";
    case LMEP_ORDER_TOO_HIGH: return "derivative order too high";
    case LMEP_DUPLICATE_NODES: return "duplicate nodes";
    default: return "unknown status";
    }
}

extern "C" const char *lmep_last_error(void) { return lmep::g_last_error; }

extern "C" int64_t lmep_launch_count(void) { return lmep::g_launches.load(); }
