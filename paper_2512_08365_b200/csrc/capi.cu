// capi.cu -- version / error strings / launch accounting for libdwb200.
#include <atomic>
#include <cstdio>
#include <cstdlib>

#include "dw_common.cuh"

namespace dw {

static thread_local int64_t g_launches = 0;
static thread_local int g_timing = 0;
constexpr int TIMING_RING = 1024;
static thread_local cudaEvent_t g_ev[2 * TIMING_RING];
static thread_local int g_nev = 0;
static thread_local double g_pending_ms = 0.0;
static thread_local int64_t g_timed = 0;  // launches timed since the last reset

void count_launch(int n) { g_launches += n; }

// fold the recorded event pairs into g_pending_ms (waits for the last one)
static void timing_drain() {
    for (int i = 0; i < g_nev; ++i) {
        float ms = 0.f;
        cudaEventSynchronize(g_ev[2 * i + 1]);
        cudaEventElapsedTime(&ms, g_ev[2 * i], g_ev[2 * i + 1]);
        g_pending_ms += ms;
    }
    g_nev = 0;
}

// Events around the attribution tile kernel (bench.py's roofline timing).
// Every launch is timed: a full ring is drained (one host wait on an event
// recorded ~1000 launches earlier) rather than dropping launches.
void timing_begin(cudaStream_t s) {
    if (!g_timing) return;
    if (g_nev >= TIMING_RING) timing_drain();
    cudaEvent_t *e = &g_ev[2 * g_nev];
    if (!e[0]) { cudaEventCreate(&e[0]); cudaEventCreate(&e[1]); }
    cudaEventRecord(e[0], s);
}
void timing_end(cudaStream_t s) {
    if (!g_timing) return;
    cudaEventRecord(g_ev[2 * g_nev + 1], s);
    ++g_nev;
    ++g_timed;
}

// Phase trace (diagnostic): with DWB200_TRACE set, trace_mark() records a
// named event on the stream; dw_trace_report() prints the time between
// consecutive marks to stderr.  Off by default (one getenv, then a branch).
static thread_local cudaEvent_t g_tev[256];
static thread_local const char *g_tname[256];
static thread_local int g_ntev = 0;
static int trace_on() {
    static int on = -1;
    if (on < 0) on = getenv("DWB200_TRACE") ? 1 : 0;
    return on;
}
void trace_mark(cudaStream_t s, const char *name) {
    if (!trace_on() || g_ntev >= 256) return;
    if (!g_tev[g_ntev]) cudaEventCreate(&g_tev[g_ntev]);
    g_tname[g_ntev] = name;
    cudaEventRecord(g_tev[g_ntev++], s);
}

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

int dw_kernel_timing(int enable) {
    dw::g_timing = enable;
    return DW_OK;
}

double dw_kernel_time_ms(int reset) {
    using namespace dw;
    timing_drain();
    const double total = g_pending_ms;
    if (reset) g_pending_ms = 0.0;
    return total;
}

int64_t dw_kernel_timed_count(int reset) {
    const int64_t n = dw::g_timed;
    if (reset) dw::g_timed = 0;
    return n;
}

void dw_trace_report(void) {
    using namespace dw;
    if (!g_ntev) return;
    cudaEventSynchronize(g_tev[g_ntev - 1]);
    for (int i = 1; i < g_ntev; ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, g_tev[i - 1], g_tev[i]);
        fprintf(stderr, "  %-28s %8.3f ms\n", g_tname[i], ms);
    }
    g_ntev = 0;
}

int64_t dw_launch_count(int reset) {
    int64_t v = dw::g_launches;
    if (reset) dw::g_launches = 0;
    return v;
}

}  // extern "C"
