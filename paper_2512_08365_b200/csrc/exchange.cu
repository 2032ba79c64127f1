// exchange.cu -- the time-window join's signature exchange (shard.py
// sharded_join) as ONE kernel over peer memory.
//
// Each rank owns a slice of one trace's operators; every operator must reach
// the rank hash(signature) % world, where all occurrences of its signature
// meet.  Instead of "pack records, sort by destination, NCCL all-to-all",
// `dw_exchange_scatter` reads the rank's operator columns once, computes each
// record's destination, and stores the packed record straight into the
// destination rank's receive buffer through a CUDA IPC mapping (NVLink /
// NVSwitch P2P stores on a multi-GPU node; plain HBM stores when ranks share
// a GPU).  Warp-aggregated atomics on a per-destination cursor give each
// warp one reservation per destination it touches; the receiver orders its
// records by global op index afterwards, as it does for the NCCL path, so
// record order inside a buffer is free.  `dw_exchange_count` is the sizing
// pass (per-destination record counts) whose counts the ranks swap before
// the receive buffers are allocated and their IPC handles shared.
#include <cstring>
#include <dlfcn.h>

#include "dw_common.cuh"

namespace dw {

constexpr int XCH_THREADS = 256;

__device__ __forceinline__ int xch_dest(int64_t sig, int world) {
    // shard.py _dest: ((sig ^ (sig >> 31)) & 0x7FFFFFFF) % world (arithmetic shift)
    return (int)(((sig ^ (sig >> 31)) & 0x7FFFFFFFLL) % world);
}

__global__ void exchange_count_kernel(const int64_t *sig, int64_t n, int world, unsigned long long *counts) {
    __shared__ unsigned long long c[DW_MAX_PEERS];
    for (int d = threadIdx.x; d < world; d += blockDim.x) c[d] = 0;
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        atomicAdd(&c[xch_dest(__ldg(sig + i), world)], 1ULL);
    __syncthreads();
    for (int d = threadIdx.x; d < world; d += blockDim.x)
        if (c[d]) atomicAdd(counts + d, c[d]);
}

struct XchCols {
    const int64_t *col[DW_XCH_MAX_WIDTH];
    int64_t *peer[DW_MAX_PEERS];  // receive buffers (IPC-mapped for other ranks)
    int64_t base[DW_MAX_PEERS];   // this rank's first record slot in each receiver's buffer
};

__global__ void exchange_scatter_kernel(XchCols x, int width, const int64_t *sig, int64_t n, int world,
                                        unsigned long long *cursor) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < n; i0 += stride) {
        const int64_t i = i0 + threadIdx.x;
        const bool live = i < n;
        const int d = live ? xch_dest(__ldg(sig + i), world) : -1;
        // warp-aggregated reservation: one atomic per destination present in the warp
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int leader = __ffs(peers) - 1;
        unsigned long long slot0 = 0;
        if (live && lane == leader) slot0 = atomicAdd(cursor + d, (unsigned long long)__popc(peers));
        slot0 = __shfl_sync(0xffffffffu, slot0, leader);
        if (!live) continue;
        const int64_t slot = x.base[d] + (int64_t)slot0 + __popc(peers & ((1u << lane) - 1u));
        int64_t *dst = x.peer[d] + slot * width;
#pragma unroll
        for (int c = 0; c < DW_XCH_MAX_WIDTH; ++c)
            if (c < width) dst[c] = __ldg(x.col[c] + i);
    }
}


// Arrival flags of the persistent mailbox (shard.Comm): after its scatter a
// sender publishes the exchange's epoch into slot [me] of every receiver's
// flag array (system-scope release, after a system fence, so its P2P record
// stores are visible first); a receiver's stream waits on the device until
// every sender's slot holds the epoch -- no host sync, no barrier.
struct XchFlags {
    unsigned long long *peer[DW_MAX_PEERS];
};

__global__ void exchange_signal_kernel(XchFlags f, int world, int me, unsigned long long epoch) {
    __threadfence_system();
    for (int d = threadIdx.x; d < world; d += blockDim.x) {
        unsigned long long *slot = f.peer[d] + me;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(slot), "l"(epoch) : "memory");
    }
}

__global__ void exchange_wait_kernel(const unsigned long long *flags, int world, unsigned long long epoch,
                                     int *timeout) {
    for (int s = threadIdx.x; s < world; s += blockDim.x) {
        const long long t0 = clock64();
        for (;;) {
            unsigned long long v;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + s) : "memory");
            if (v >= epoch) break;
            if (clock64() - t0 > (long long)40000000000LL) {  // ~20 s at 2 GHz: a peer never signalled
                atomicExch(timeout, 1);
                break;
            }
            __nanosleep(256);
        }
    }
    __threadfence_system();
}

}  // namespace dw

using namespace dw;

extern "C" {

int dw_exchange_count(const int64_t *d_sig, int64_t n, int32_t world, uint64_t *d_counts, dw_stream_t stream) {
    if (n < 0 || world < 1 || world > DW_MAX_PEERS || !d_counts || (n && !d_sig)) return DW_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(d_counts, 0, sizeof(uint64_t) * world, s);
    if (n) {
        exchange_count_kernel<<<(unsigned)std::min<int64_t>(num_sms() * 8, ceil_div(n, XCH_THREADS)), XCH_THREADS,
                                0, s>>>(d_sig, n, world, (unsigned long long *)d_counts);
        count_launch();
    }
    DW_CHECK_LAUNCH();
    return DW_OK;
}

int dw_exchange_scatter(const int64_t *const *cols, int32_t width, const int64_t *d_sig, int64_t n, int32_t world,
                        int64_t *const *d_peer, const int64_t *base, uint64_t *d_cursor, dw_stream_t stream) {
    if (n < 0 || world < 1 || world > DW_MAX_PEERS || width < 1 || width > DW_XCH_MAX_WIDTH || !d_cursor ||
        !cols || !d_peer || !base || (n && !d_sig))
        return DW_E_ARG;
    XchCols x{};
    for (int c = 0; c < width; ++c) {
        if (n && !cols[c]) return DW_E_ARG;
        x.col[c] = cols[c];
    }
    for (int d = 0; d < world; ++d) {
        x.peer[d] = d_peer[d];
        x.base[d] = base[d];
    }
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(d_cursor, 0, sizeof(uint64_t) * world, s);
    if (n) {
        exchange_scatter_kernel<<<(unsigned)std::min<int64_t>(num_sms() * 8, ceil_div(n, XCH_THREADS)),
                                  XCH_THREADS, 0, s>>>(x, width, d_sig, n, world, (unsigned long long *)d_cursor);
        count_launch();
    }
    DW_CHECK_LAUNCH();
    return DW_OK;
}


int dw_exchange_signal(uint64_t *const *d_peer_flags, int32_t world, int32_t me, uint64_t epoch,
                       dw_stream_t stream) {
    if (world < 1 || world > DW_MAX_PEERS || me < 0 || me >= world || !d_peer_flags) return DW_E_ARG;
    XchFlags f{};
    for (int d = 0; d < world; ++d) {
        if (!d_peer_flags[d]) return DW_E_ARG;
        f.peer[d] = (unsigned long long *)d_peer_flags[d];
    }
    exchange_signal_kernel<<<1, 64, 0, (cudaStream_t)stream>>>(f, world, me, (unsigned long long)epoch);
    count_launch();
    DW_CHECK_LAUNCH();
    return DW_OK;
}

int dw_exchange_wait(const uint64_t *d_flags, int32_t world, uint64_t epoch, int32_t *d_timeout,
                     dw_stream_t stream) {
    if (world < 1 || world > DW_MAX_PEERS || !d_flags || !d_timeout) return DW_E_ARG;
    exchange_wait_kernel<<<1, 64, 0, (cudaStream_t)stream>>>((const unsigned long long *)d_flags, world,
                                                             (unsigned long long)epoch, (int *)d_timeout);
    count_launch();
    DW_CHECK_LAUNCH();
    return DW_OK;
}

// The handle names a whole allocation; buffers from a caching allocator sit
// inside one, so the handle carries the buffer's offset from the allocation
// base (driver cuMemGetAddressRange, looked up at run time: libdwb200 links
// only the runtime).
typedef int (*GetRangeFn)(unsigned long long *, size_t *, unsigned long long);

static GetRangeFn get_range() {
    static GetRangeFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *lib = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
        if (lib) fn = (GetRangeFn)dlsym(lib, "cuMemGetAddressRange_v2");
    }
    return fn;
}

int dw_ipc_handle(const void *d_ptr, void *handle_out, int64_t *offset_out) {
    if (!d_ptr || !handle_out || !offset_out) return DW_E_ARG;
    GetRangeFn range = get_range();
    if (!range) return DW_E_CUDA;
    unsigned long long base = 0;
    size_t size = 0;
    if (range(&base, &size, (unsigned long long)(uintptr_t)d_ptr) != 0) return DW_E_CUDA;
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base) != cudaSuccess) return DW_E_CUDA;
    memcpy(handle_out, &h, sizeof(h));
    *offset_out = (int64_t)((uintptr_t)d_ptr - (uintptr_t)base);
    return DW_OK;
}

int dw_ipc_open(const void *handle, void **d_ptr_out) {
    if (!handle || !d_ptr_out) return DW_E_ARG;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    if (cudaIpcOpenMemHandle(d_ptr_out, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return DW_E_CUDA;
    return DW_OK;
}

int dw_ipc_close(void *d_ptr) {
    if (!d_ptr) return DW_E_ARG;
    return cudaIpcCloseMemHandle(d_ptr) == cudaSuccess ? DW_OK : DW_E_CUDA;
}

}  // extern "C"
