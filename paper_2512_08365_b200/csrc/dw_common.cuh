// dw_common.cuh -- shared device helpers for libdwb200 (sm_100a).
//
//  * exact fixed-point accumulation (int128) used for long intervals and large
//    reductions -- bit-identical to oracle/dw_oracle.c's fx_from_double /
//    fx_to_double;
//  * CPython-3.12 sum() (Neumaier) for reference-faithful short sums;
//  * 1-D TMA (cp.async.bulk) + mbarrier wrappers;
//  * launch accounting and status-block layout.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/dwb200.h"

namespace dw {

typedef __int128 i128;
typedef unsigned __int128 u128;

constexpr int FX_TERM_BITS = 40;   // integrand terms, W*us
constexpr int FX_JOULE_BITS = 64;  // sums of joules
constexpr double US_PER_S = 1000000.0;
constexpr int64_t NONE = INT64_MAX;  // "no index" inside the status block

// ---------------------------------------------------------------- status block
// Lives at the head of every workspace.  Indices are kept as INT64_MAX while
// running (atomicMin) and translated to -1 by dw_status().
struct DevStatus {
    unsigned long long bad_index[DW_MAX_SETS];
    unsigned long long unsorted_index[DW_MAX_SETS];
    unsigned long long order_index;
    unsigned long long long_count;
    double totals[4];
    unsigned long long pad[4];
};
static_assert(sizeof(DevStatus) <= 256, "status block");
constexpr size_t STATUS_BYTES = 256;

// ---------------------------------------------------------------- fixed point
__host__ __device__ __forceinline__ i128 fx_from_double(double x, int scale) {
    if (x == 0.0) return 0;
#ifdef __CUDA_ARCH__
    uint64_t bits = (uint64_t)__double_as_longlong(x);
#else
    uint64_t bits;
    __builtin_memcpy(&bits, &x, 8);
#endif
    int neg = (int)(bits >> 63);
    int e = (int)((bits >> 52) & 0x7ff);
    uint64_t m = bits & 0xfffffffffffffULL;
    if (e == 0) e = 1; else m |= 1ULL << 52;
    int sh = e - 1075 + scale;
    i128 v;
    if (sh >= 0) {
        v = (i128)m << sh;
    } else {
        int r = -sh;
        if (r >= 64) {
            v = 0;
        } else {
            uint64_t q = m >> r;
            uint64_t rem = m & ((1ULL << r) - 1);
            uint64_t half = 1ULL << (r - 1);
            if (rem > half || (rem == half && (q & 1))) q++;
            v = (i128)q;
        }
    }
    return neg ? -v : v;
}

__host__ __device__ __forceinline__ int clz64(uint64_t x) {
#ifdef __CUDA_ARCH__
    return __clzll((long long)x);
#else
    return __builtin_clzll(x);
#endif
}

__host__ __device__ __forceinline__ double fx_to_double(i128 v, int scale) {
    int neg = v < 0;
    u128 u = neg ? (u128)(-v) : (u128)v;
    double r;
    if ((u >> 53) == 0) {
        r = (double)(uint64_t)u;
    } else {
        uint64_t hi = (uint64_t)(u >> 64), lo = (uint64_t)u;
        int len = hi ? 128 - clz64(hi) : 64 - clz64(lo);
        int drop = len - 53;
        u128 q = u >> drop;
        u128 rem = u & ((((u128)1) << drop) - 1);
        u128 half = ((u128)1) << (drop - 1);
        if (rem > half || (rem == half && (q & 1))) q++;
        r = ldexp((double)(uint64_t)q, drop);
    }
    r = ldexp(r, -scale);
    return neg ? -r : r;
}

__host__ __device__ __forceinline__ i128 q_term(double x) { return fx_from_double(x, FX_TERM_BITS); }

// q_term for |x| < 2^23 (|x * 2^40| < 2^63) in two instructions: the scaling
// by 2^40 is exact and cvt.rni rounds half to even, as fx_from_double does.
constexpr double Q40_FAST_LIMIT = 8388608.0;  // 2^23 W*us
__device__ __forceinline__ bool q40_fast(double x, long long &q) {
    if (!(fabs(x) < Q40_FAST_LIMIT)) return false;
    q = __double2ll_rn(__dmul_rn(x, 1099511627776.0));
    return true;
}
// fx_from_double(x, FX_JOULE_BITS) with the int128 shifts only for |x| >= 2^10
// J: below 0.5 J the scaling by 2^64 is exact and cvt.rni rounds half to even
// (values under 2^-11 J round to 0 either way); in [0.5, 2^10) J every x is a
// multiple of 2^-53, so x * 2^53 converts exactly and the shift by 11 is the
// rest of the scale.
__device__ __forceinline__ i128 fx_joules(double x) {
    const double a = fabs(x);
    if (a < 0.5) return (i128)__double2ll_rn(__dmul_rn(x, 18446744073709551616.0));
    if (a < 1024.0) return (i128)__double2ll_rn(__dmul_rn(x, 9007199254740992.0)) * 2048;  // (no signed shift)
    return fx_from_double(x, FX_JOULE_BITS);
}
__device__ __forceinline__ i128 q40(double x) {
    long long q;
    return q40_fast(x, q) ? (i128)q : q_term(x);
}

__host__ __device__ __forceinline__ double term_fx_to_joules(i128 v) {
    return fx_to_double(v, FX_TERM_BITS) / US_PER_S;
}

// int128 split for shuffles / storage
struct I128Parts { uint64_t lo, hi; };
__device__ __forceinline__ I128Parts split(i128 v) {
    u128 u = (u128)v;
    return {(uint64_t)u, (uint64_t)(u >> 64)};
}
__device__ __forceinline__ i128 join(uint64_t lo, uint64_t hi) {
    return (i128)(((u128)hi << 64) | (u128)lo);
}

__device__ __forceinline__ i128 warp_sum_i128(i128 v) {
    I128Parts p = split(v);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t lo = __shfl_xor_sync(0xffffffffu, p.lo, o);
        uint64_t hi = __shfl_xor_sync(0xffffffffu, p.hi, o);
        i128 s = join(p.lo, p.hi) + join(lo, hi);
        p = split(s);
    }
    return join(p.lo, p.hi);
}

// ---------------------------------------------------------------- python sum()
// CPython >= 3.12 builtin sum over floats (Neumaier); reference sums
// (subgraph_joules energy.py:277, report detect.py:267) go through it.
struct PySum {
    double f, c;
    int64_t n;
    __host__ __device__ __forceinline__ PySum() : f(0.0), c(0.0), n(0) {}
    __host__ __device__ __forceinline__ void add(double x) {
        if (n++ == 0) { f = x; c = 0.0; return; }
        double t = __dadd_rn_(f, x);
        if (fabs(f) >= fabs(x)) c = __dadd_rn_(c, __dadd_rn_(__dsub_rn_(f, t), x));
        else c = __dadd_rn_(c, __dadd_rn_(__dsub_rn_(x, t), f));
        f = t;
    }
    __host__ __device__ __forceinline__ double result() const {
        if (n == 0) return 0.0;
        double r = f;
        if (c != 0.0 && isfinite(c)) r = __dadd_rn_(r, c);
        return r;
    }
    // explicit round-to-nearest ops; no FMA contraction possible
    __host__ __device__ static __forceinline__ double __dadd_rn_(double a, double b) {
#ifdef __CUDA_ARCH__
        return __dadd_rn(a, b);
#else
        return a + b;
#endif
    }
    __host__ __device__ static __forceinline__ double __dsub_rn_(double a, double b) {
#ifdef __CUDA_ARCH__
        return __dsub_rn(a, b);
#else
        return a - b;
#endif
    }
};

// ---------------------------------------------------------------- 1-D TMA
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// cp.async.bulk global -> shared, completion via mbarrier transaction bytes.
// dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- misc
__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

__device__ __forceinline__ void atomic_min_index(unsigned long long *p, int64_t v) {
    atomicMin(p, (unsigned long long)v);
}

// host-side launch accounting (bench.py gpu_launches)
void count_launch(int n = 1);
void timing_begin(cudaStream_t s);
void timing_end(cudaStream_t s);
void trace_mark(cudaStream_t s, const char *name);
int num_sms();

}  // namespace dw

#define DW_CHECK_LAUNCH()                                      \
    do {                                                       \
        cudaError_t e__ = cudaGetLastError();                  \
        if (e__ != cudaSuccess) return DW_E_CUDA;              \
    } while (0)
