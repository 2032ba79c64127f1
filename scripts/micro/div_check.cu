// Check the fast exact quotient used for the trapezoid frac (attribute.cu
// div_u32) against IEEE __ddiv_rn: exhaustive for den <= 4096, random pairs beyond.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ double div_u32(uint32_t num, uint32_t den) {
    const double b = (double)den, a = (double)num;
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(b));
    double e = __fma_rn(-b, y, 1.0);
    y = __fma_rn(y, e, y);
    e = __fma_rn(-b, y, 1.0);
    y = __fma_rn(y, e, y);
    double q = __dmul_rn(a, y);
    double r = __fma_rn(-q, b, a);
    return __fma_rn(r, y, q);
}
__global__ void exhaustive(unsigned long long *bad, uint32_t dmax) {
    uint32_t den = blockIdx.x + 1;
    if (den > dmax) return;
    for (uint32_t num = threadIdx.x; num <= den; num += blockDim.x)
        if (__double_as_longlong(div_u32(num, den)) != __double_as_longlong(__ddiv_rn((double)num, (double)den)))
            atomicAdd(bad, 1ULL);
}
__device__ __forceinline__ uint64_t mix(uint64_t x) { x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33; return x; }
__global__ void random_pairs(unsigned long long *bad, uint64_t n, uint64_t seed) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t h = mix(i ^ seed);
        int bits = 1 + (int)(h & 31);
        uint32_t den = (uint32_t)((h >> 8) & ((1ULL << bits) - 1)) | 1u;
        den = den ? den : 1u;
        uint32_t num = (uint32_t)(mix(h) % ((uint64_t)den + 1));
        if (__double_as_longlong(div_u32(num, den)) != __double_as_longlong(__ddiv_rn((double)num, (double)den)))
            atomicAdd(bad, 1ULL);
    }
}
int main() {
    unsigned long long *d, h = 0; cudaMalloc(&d, 8); cudaMemset(d, 0, 8);
    exhaustive<<<4096, 256>>>(d, 4096);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("exhaustive den<=4096: %llu mismatches\n", h);
    cudaMemset(d, 0, 8);
    random_pairs<<<148 * 8, 256>>>(d, 4000000000ULL, 12345);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("random 4e9 pairs (den < 2^32): %llu mismatches\n", h);
    return 0;
}
