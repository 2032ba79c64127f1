// capi.cu -- version / error strings / launch accounting for libdwb200.
#include <atomic>

#include "dw_common.cuh"

namespace dw {

static thread_local int64_t g_launches = 0;

void count_launch(int n) { g_launches += n; }

int num_sms() {
    static thread_local int cached_dev = -1, cached_sms = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != cached_dev) {
        cudaDeviceGetAttribute(&cached_sms, cudaDevAttrMultiProcessorCount, dev);
        cached_dev = dev;
    }
    return cached_sms > 0 ? cached_sms : 148;
}

}  // namespace dw

extern "C" {

const char *dw_version(void) { return "dwb200 0.1.0 sm_100a"; }

const char *dw_error_string(int code) {
    switch (code) {
        case DW_OK: return "ok";
        case DW_E_REVERSED: return "interval end precedes start";
        case DW_E_SPAN: return "interval outside signal span";
        case DW_E_EMPTY: return "empty power signal";
        case DW_E_ORDER: return "power samples must be strictly increasing in timestamp";
        case DW_E_ARG: return "invalid argument";
        case DW_E_CUDA: return "CUDA error";
        case DW_E_WORKSPACE: return "workspace too small";
        case DW_E_UNSORTED: return "interval set flagged sorted is not sorted by start";
        default: return "unknown error";
    }
}

int64_t dw_launch_count(int reset) {
    int64_t v = dw::g_launches;
    if (reset) dw::g_launches = 0;
    return v;
}

}  // extern "C"
