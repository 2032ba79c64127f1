// Micro-benchmark: CUB onesweep radix sort with wider digits (custom policy
// hub) for the join's (id, index) sort: 1e8 u32/u32 pairs, 21-bit ids.
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdint>

template <typename KeyT, typename ValueT, typename OffsetT, int BITS, int ITEMS, int THREADS>
struct WideHub {
    using base = cub::detail::radix::policy_hub<KeyT, ValueT, OffsetT>;
    struct Policy1000 : cub::ChainedPolicy<1000, Policy1000, Policy1000> {
        using B = typename base::Policy1000;
        static constexpr bool ONESWEEP = true;
        static constexpr int ONESWEEP_RADIX_BITS = BITS;
        using HistogramPolicy = cub::AgentRadixSortHistogramPolicy<128, 16, 1, KeyT, BITS>;
        using ExclusiveSumPolicy = cub::AgentRadixSortExclusiveSumPolicy<256, BITS>;
        using OnesweepPolicy = cub::AgentRadixSortOnesweepPolicy<THREADS, ITEMS, KeyT, 1, cub::RADIX_RANK_MATCH_EARLY_COUNTS_ANY,
                                                                 cub::BLOCK_SCAN_RAKING_MEMOIZE, cub::RADIX_SORT_STORE_DIRECT, BITS>;
        using ScanPolicy = typename B::ScanPolicy;
        using DownsweepPolicy = typename B::DownsweepPolicy;
        using AltDownsweepPolicy = typename B::AltDownsweepPolicy;
        using UpsweepPolicy = typename B::UpsweepPolicy;
        using AltUpsweepPolicy = typename B::AltUpsweepPolicy;
        using SingleTilePolicy = typename B::SingleTilePolicy;
        using SegmentedPolicy = typename B::SegmentedPolicy;
        using AltSegmentedPolicy = typename B::AltSegmentedPolicy;
    };
    using MaxPolicy = Policy1000;
};

__global__ void fill(uint32_t *k, uint32_t *v, int n, int bits) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t x = (uint64_t)i * 0x9E3779B97F4A7C15ULL;
    x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ULL; x ^= x >> 32;
    k[i] = (uint32_t)(x & ((1u << bits) - 1));
    v[i] = i;
}

template <int BITS, int ITEMS, int THREADS>
void run(uint32_t *k0, uint32_t *v0, uint32_t *k1, uint32_t *v1, uint32_t *kk, uint32_t *vv, int n, int bits) {
    using D = cub::DispatchRadixSort<false, uint32_t, uint32_t, int, WideHub<uint32_t, uint32_t, int, BITS, ITEMS, THREADS>>;
    size_t t = 0;
    cub::DoubleBuffer<uint32_t> dk(k1, kk), dv(v1, vv);
    D::Dispatch(nullptr, t, dk, dv, n, 0, bits, false, 0);
    void *tmp; cudaMalloc(&tmp, t);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemcpy(k1, k0, 4ull * n, cudaMemcpyDeviceToDevice);
        cudaMemcpy(v1, v0, 4ull * n, cudaMemcpyDeviceToDevice);
        cub::DoubleBuffer<uint32_t> dk2(k1, kk), dv2(v1, vv);
        float ms;
        cudaEventRecord(a);
        cudaError_t e = D::Dispatch(tmp, t, dk2, dv2, n, 0, bits, false, 0);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("BITS=%d ITEMS=%d THREADS=%d: %.3f ms (%s)\n", BITS, ITEMS, THREADS, ms, cudaGetErrorString(e ? e : cudaGetLastError()));
    }
    cudaFree(tmp);
}

int main() {
    const int n = 100000000, bits = 21;
    uint32_t *k0, *v0, *k1, *v1, *kk, *vv;
    cudaMalloc(&k0, 4ull * n); cudaMalloc(&v0, 4ull * n); cudaMalloc(&k1, 4ull * n); cudaMalloc(&v1, 4ull * n);
    cudaMalloc(&kk, 4ull * n); cudaMalloc(&vv, 4ull * n);
    fill<<<(n + 255) / 256, 256>>>(k0, v0, n, bits);
    size_t t = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t, k0, k1, v0, v1, n, 0, bits);
    void *tmp; cudaMalloc(&tmp, t);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
        cudaEventRecord(a);
        cub::DeviceRadixSort::SortPairs(tmp, t, k0, k1, v0, v1, n, 0, bits);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("default SortPairs: %.3f ms\n", ms);
    }
    run<8, 23, 384>(k0, v0, k1, v1, kk, vv, n, bits);
    run<11, 16, 96>(k0, v0, k1, v1, kk, vv, n, bits);
    run<11, 32, 96>(k0, v0, k1, v1, kk, vv, n, bits);
    run<11, 32, 64>(k0, v0, k1, v1, kk, vv, n, bits);
    run<11, 48, 64>(k0, v0, k1, v1, kk, vv, n, bits);
    return 0;
}
