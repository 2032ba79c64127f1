// Micro-benchmark: CUB radix sort variants for the join's grouping sort
// (1e8 elements, ~20-bit ids).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 sort_bench.cu
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void fill(uint64_t *k64, uint32_t *k32, uint32_t *v32, int n, int bits) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t x = (uint64_t)i * 0x9E3779B97F4A7C15ULL;
    x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ULL; x ^= x >> 32;
    uint32_t d = (uint32_t)(x & ((1u << bits) - 1));
    k64[i] = ((uint64_t)d << 32) | (uint32_t)i;
    k32[i] = d;
    v32[i] = i;
}

int main() {
    const int n = 100000000, bits = 20;
    uint64_t *k64, *o64; uint32_t *k32, *o32, *v32, *w32;
    cudaMalloc(&k64, 8ull * n); cudaMalloc(&o64, 8ull * n);
    cudaMalloc(&k32, 4ull * n); cudaMalloc(&o32, 4ull * n);
    cudaMalloc(&v32, 4ull * n); cudaMalloc(&w32, 4ull * n);
    fill<<<(n + 255) / 256, 256>>>(k64, k32, v32, n, bits);
    size_t t1 = 0, t2 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, t1, k64, o64, n, 32, 32 + bits);
    cub::DeviceRadixSort::SortPairs(nullptr, t2, k32, o32, v32, w32, n, 0, bits);
    void *tmp; cudaMalloc(&tmp, t1 > t2 ? t1 : t2);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        float ms;
        cudaEventRecord(a);
        cub::DeviceRadixSort::SortKeys(tmp, t1, k64, o64, n, 32, 32 + bits);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("SortKeys u64 bits[32,%d): %.3f ms\n", 32 + bits, ms);
        cudaEventRecord(a);
        cub::DeviceRadixSort::SortPairs(tmp, t2, k32, o32, v32, w32, n, 0, bits);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("SortPairs u32/u32 bits[0,%d): %.3f ms\n", bits, ms);
        cudaEventRecord(a);
        cudaMemcpy(o64, k64, 8ull * n, cudaMemcpyDeviceToDevice);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("copy 800MB: %.3f ms (%.1f GB/s)\n", ms, 1.6e9 / ms / 1e6);
    }
    return 0;
}
