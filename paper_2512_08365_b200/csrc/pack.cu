// pack.cu -- device decode of the packed columnar trace format (ingestion,
// SURVEY.md 8(a) a1 / 8(f) 1).
//
// On the host (and on disk, shard.py / columns.py) a trace keeps its sorted
// timestamp columns as 32-bit deltas and its interval ends as 32-bit
// durations: ts 8 -> 4 bytes per sample, intervals 16 -> 8 bytes.  The
// host->HBM copy is what bounds the end-to-end path (PCIe), so this cuts the
// bytes that cross it by ~30 %; the decode here is one CUB scan per column
// (HBM-bound) plus a fused start + duration pass.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "dw_common.cuh"

namespace dw {

struct DeltaAt {  // value i of the scan input: base + d[0] at 0, d[i] after
    const uint32_t *d;
    int64_t base;
    __host__ __device__ int64_t operator()(int64_t i) const { return i == 0 ? base + (int64_t)d[0] : (int64_t)d[i]; }
};

__global__ void add_duration_kernel(const int64_t *start, const uint32_t *dur, int64_t n, int64_t *end) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        end[i] = __ldcs(start + i) + (int64_t)__ldcs(dur + i);
}

static size_t scan_bytes(int64_t n) {
    size_t b = 0;
    auto it = thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0), DeltaAt{nullptr, 0});
    cub::DeviceScan::InclusiveSum(nullptr, b, it, (int64_t *)nullptr, (int)std::max<int64_t>(n, 1));
    return b;
}

}  // namespace dw

using namespace dw;

extern "C" {

size_t dw_unpack_workspace_size(int64_t n) { return scan_bytes(n) + 256; }

int dw_unpack_deltas(const uint32_t *d_delta, int64_t n, int64_t base, int64_t *d_out, const uint32_t *d_dur,
                     int64_t *d_end, void *d_workspace, size_t workspace_bytes, dw_stream_t stream) {
    if (n < 0 || (n && (!d_delta || !d_out)) || (d_dur && !d_end) || n >= ((int64_t)1 << 31)) return DW_E_ARG;
    if (n == 0) return DW_OK;
    if (!d_workspace || workspace_bytes < dw_unpack_workspace_size(n)) return DW_E_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    auto it = thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0), DeltaAt{d_delta, base});
    size_t b = workspace_bytes;
    cub::DeviceScan::InclusiveSum(d_workspace, b, it, d_out, (int)n, s);
    count_launch(2);
    if (d_dur) {
        add_duration_kernel<<<(unsigned)std::min<int64_t>(num_sms() * 8, ceil_div(n, 256)), 256, 0, s>>>(
            d_out, d_dur, n, d_end);
        count_launch();
    }
    DW_CHECK_LAUNCH();
    return DW_OK;
}

}  // extern "C"
