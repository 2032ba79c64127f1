// Check the decimal decode (pack.cu decimal_decode_kernel): m / 10^p by a
// correctly rounded reciprocal plus Markstein's final FMA step, against IEEE
// __ddiv_rn -- exhaustive over every m < 2^30 for every p in 0..22.
#include <cstdio>
#include <cstdint>
__constant__ double POW10[23] = {1e0, 1e1, 1e2, 1e3, 1e4, 1e5, 1e6, 1e7, 1e8, 1e9, 1e10, 1e11,
                                 1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
__constant__ double RCP10[23] = {1.0, 0.1, 0.01, 0.001, 0.0001, 1e-05, 1e-06, 1e-07, 1e-08, 1e-09, 1e-10, 1e-11, 1e-12, 1e-13, 1e-14, 1e-15, 1e-16, 1e-17, 1e-18, 1e-19, 1e-20, 1e-21, 1e-22};
__device__ __forceinline__ double dec(double m, int p) {
    const double y = RCP10[p], d = POW10[p];
    const double q = __dmul_rn(m, y);
    const double r = __fma_rn(-q, d, m);
    return __fma_rn(r, y, q);
}
__global__ void check(unsigned long long *bad, int p) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    unsigned long long nb = 0;
    for (uint64_t m = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; m < (1ULL << 30); m += stride)
        nb += __double_as_longlong(dec((double)m, p)) != __double_as_longlong(__ddiv_rn((double)m, POW10[p]));
    if (nb) atomicAdd(bad, nb);
}
int main() {
    unsigned long long *d, h, total = 0;
    cudaMalloc(&d, 8);
    for (int p = 0; p < 23; ++p) {
        cudaMemset(d, 0, 8);
        check<<<148 * 16, 256>>>(d, p);
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        total += h;
        printf("p=%2d mismatches %llu\n", p, h);
    }
    printf("total mismatches %llu over 23 x 2^30\n", total);
    return 0;
}
