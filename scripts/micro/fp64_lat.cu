// FP64 latency / throughput microbenchmark (dependent chains, clock64)
#include <cstdio>
#include <cstdint>
__global__ void lat_dadd(double *out, double x, int n, long long *cyc) {
    double a = x, b = x * 0.5;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { a = __dadd_rn(a, b); }
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_dmul(double *out, double x, int n, long long *cyc) {
    double a = x, b = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { a = __dmul_rn(a, b); }
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_ddiv(double *out, double x, int n, long long *cyc) {
    double a = x + threadIdx.x, b = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { a = __ddiv_rn(b, a) + 1.0; }
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_i2d(double *out, int x, int n, long long *cyc) {
    double a = 0; int v = x + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { a = (double)v; v = (int)__double_as_longlong(a) ^ i; }
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// throughput: 8 independent chains per thread, many warps
__global__ void thr_dadd(double *out, double x, int n) {
    double a[8]; for (int k = 0; k < 8; ++k) a[k] = x + k;
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = __dadd_rn(a[k], 1e-3);
    double s = 0; for (int k = 0; k < 8; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void thr_i2d(double *out, int x, int n) {
    double a[8]; int v[8]; for (int k = 0; k < 8; ++k) { v[k] = x + k + threadIdx.x; a[k] = 0; }
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) { a[k] += (double)(v[k] + i); }
    double s = 0; for (int k = 0; k < 8; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    double *d; long long *c; cudaMalloc(&d, 1 << 26); cudaMalloc(&c, 8);
    long long h; int n = 4096;
    lat_dadd<<<1, 32>>>(d, 1.0, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("DADD lat %.2f cyc\n", (double)h / n);
    lat_dmul<<<1, 32>>>(d, 1.0, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("DMUL lat %.2f cyc\n", (double)h / n);
    lat_ddiv<<<1, 32>>>(d, 1.0, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("DDIV+DADD lat %.2f cyc\n", (double)h / n);
    lat_i2d<<<1, 32>>>(d, 1, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("I2F.F64 (+ALU) lat %.2f cyc\n", (double)h / n);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
    int blocks = 148 * 8, thr = 256, m = 4096;
    thr_dadd<<<blocks, thr>>>(d, 1.0, m); cudaEventRecord(e0); thr_dadd<<<blocks, thr>>>(d, 1.0, m); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("DADD throughput %.1f Gop/s = %.1f /clk/SM @1.965GHz\n", (double)blocks*thr*m*8/ms/1e6, (double)blocks*thr*m*8/(ms*1e-3)/148/1.965e9);
    thr_i2d<<<blocks, thr>>>(d, 1, m); cudaEventRecord(e0); thr_i2d<<<blocks, thr>>>(d, 1, m); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("I2F.F64+DADD throughput %.1f Gop/s = %.1f /clk/SM\n", (double)blocks*thr*m*8/ms/1e6, (double)blocks*thr*m*8/(ms*1e-3)/148/1.965e9);
    return 0;
}
