// pack.cu -- device decode of the packed columnar trace format (ingestion,
// SURVEY.md 8(a) a1 / 8(f) 1).
//
// On the host (and on disk, shard.py / columns.py) a trace keeps its sorted
// timestamp columns as 32-bit deltas and its interval ends as 32-bit
// durations: ts 8 -> 4 bytes per sample, intervals 16 -> 8 bytes.  The
// host->HBM copy is what bounds the end-to-end path (PCIe), so this cuts the
// bytes that cross it by ~30 %; the decode here is one reduce-then-scan per
// column (HBM-bound: the packed fields are read twice, the int64 column
// written once) with the interval ends written by the same pass.

#include "dw_common.cuh"

namespace dw {

template <typename T>
struct DeltaAt {  // value i of the scan input: base at 0, bias + d[i] after
    const T *d;
    int64_t base, bias;
    __host__ __device__ int64_t operator()(int64_t i) const { return i == 0 ? base : bias + (int64_t)d[i]; }
};

// value i of a bit-packed delta column: base at 0, bias + the width-bit field
// i after (fields little-endian in 32-bit words; the words array carries one
// padding word so the 64-bit window never reads past it)
struct BitsAt {
    const uint32_t *w;
    int width;
    int64_t base, bias;
    __host__ __device__ int64_t operator()(int64_t i) const {
        if (i == 0) return base;
        const int64_t bit = i * (int64_t)width;
        const int64_t k = bit >> 5;
        const uint64_t win = (uint64_t)w[k] | ((uint64_t)w[k + 1] << 32);
        const uint64_t mask = width == 64 ? ~0ULL : ((1ULL << width) - 1ULL);
        return bias + (int64_t)((win >> (bit & 31)) & mask);
    }
};

// end[i] = start[i] + bias + field i (bit-packed durations; field 0 counts)
__global__ void add_bits_duration_kernel(const int64_t *start, const uint32_t *w, int width, int64_t bias, int64_t n,
                                         int64_t *end) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const uint64_t mask = (1ULL << width) - 1ULL;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const int64_t bit = i * (int64_t)width;
        const int64_t k = bit >> 5;
        const uint64_t win = (uint64_t)__ldg(w + k) | ((uint64_t)__ldg(w + k + 1) << 32);
        end[i] = __ldcs(start + i) + bias + (int64_t)((win >> (bit & 31)) & mask);
    }
}

template <typename T>
__global__ void add_duration_kernel(const int64_t *start, const T *dur, int64_t n, int64_t *end) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        end[i] = __ldcs(start + i) + (int64_t)__ldcs(dur + i);
}

// ---- delta-column scan: out[i] = V(0) + ... + V(i), V = DeltaAt / BitsAt,
// optionally end[i] = out[i] + E(i).  Three passes over blocks of US_B
// elements: the block sums of V, their exclusive scan (rep_scan_kernel, one
// block), then each block again -- V in registers (US_I consecutive
// elements per thread), the thread and block prefixes, the results through a
// padded shared-memory tile so the int64 stores are coalesced.
constexpr int US_T = 256, US_I = 16, US_B = US_T * US_I;

struct NoEnd {
    __device__ int64_t operator()(int64_t) const { return 0; }
};
template <typename T>
struct DurAt {  // interval end = start + d[i]
    const T *d;
    __device__ int64_t operator()(int64_t i) const { return (int64_t)d[i]; }
};
struct BitsDurAt {  // interval end = start + bias + field i (field 0 counts)
    const uint32_t *w;
    int width;
    int64_t bias;
    __device__ int64_t operator()(int64_t i) const {
        const int64_t bit = i * (int64_t)width;
        const int64_t k = bit >> 5;
        const uint64_t win = (uint64_t)__ldg(w + k) | ((uint64_t)__ldg(w + k + 1) << 32);
        return bias + (int64_t)((win >> (bit & 31)) & ((1ULL << width) - 1ULL));
    }
};

__device__ __forceinline__ int64_t block_sum_i64(int64_t v, int64_t *ws) {  // US_T threads
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
    __syncthreads();
    int64_t t = 0;
#pragma unroll
    for (int w = 0; w < US_T / 32; ++w) t += ws[w];
    return t;
}

// (both passes persistent: a few resident blocks per SM walk the chunks)
template <typename V>
__global__ void __launch_bounds__(US_T) us_sum_kernel(V val, int64_t n, int64_t nb, unsigned long long *bsum) {
    __shared__ int64_t ws[2][US_T / 32];
    int par = 0;
    for (int64_t b = blockIdx.x; b < nb; b += gridDim.x, par ^= 1) {
        const int64_t i0 = b * (int64_t)US_B;
        int64_t s = 0;
#pragma unroll 4
        for (int k = threadIdx.x; k < US_B; k += US_T)  // striped: coalesced field reads
            if (i0 + k < n) s += val(i0 + k);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if ((threadIdx.x & 31) == 0) ws[par][threadIdx.x >> 5] = s;
        __syncthreads();  // (double-buffered: one barrier per chunk)
        if (threadIdx.x == 0) {
            int64_t t = 0;
#pragma unroll
            for (int w = 0; w < US_T / 32; ++w) t += ws[par][w];
            bsum[b] = (unsigned long long)t;
        }
    }
}

template <typename V, typename E>
__global__ void __launch_bounds__(US_T) us_write_kernel(V val, E endv, int64_t n, int64_t nb,
                                                        const unsigned long long *bpre, int64_t *out, int64_t *end) {
    __shared__ int64_t tile[US_B + US_B / US_I];  // one pad per thread row: conflict-free 8-byte access
    __shared__ int64_t wt[US_T / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const int64_t i0 = b * (int64_t)US_B;
    const int64_t r0 = i0 + (int64_t)threadIdx.x * US_I;  // this thread's first element
    int64_t x[US_I];
    int64_t run = 0;
#pragma unroll
    for (int j = 0; j < US_I; ++j) {
        run += r0 + j < n ? val(r0 + j) : 0;
        x[j] = run;
    }
    int64_t inc = run;  // block-exclusive prefix of the thread totals
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) wt[warp] = inc;
    __syncthreads();
    int64_t pre = (int64_t)bpre[b] + inc - run;
    for (int w = 0; w < warp; ++w) pre += wt[w];
    int64_t *row = tile + threadIdx.x * (US_I + 1);
#pragma unroll
    for (int j = 0; j < US_I; ++j) row[j] = pre + x[j];
    __syncthreads();
    for (int k = threadIdx.x; k < US_B; k += US_T) {
        const int64_t i = i0 + k;
        if (i >= n) break;
        const int64_t v = tile[k + k / US_I];
        __stcs(out + i, v);
        if (end) __stcs(end + i, v + endv(i));
    }
    __syncthreads();  // the tile and wt are reused by the next chunk
    }
}

__global__ void __launch_bounds__(1024) rep_scan_kernel(unsigned long long *bsum, int64_t nb);

template <typename V, typename E>
static void unpack_scan(V val, E endv, int64_t n, int64_t *out, int64_t *end, void *ws, cudaStream_t s) {
    const int64_t nb = ceil_div(n, US_B);
    unsigned long long *bsum = (unsigned long long *)ws;
    const unsigned grid = (unsigned)nb;  // one chunk per block (measured: persistent blocks are slower here)
    us_sum_kernel<V><<<grid, US_T, 0, s>>>(val, n, nb, bsum);
    rep_scan_kernel<<<1, 1024, 0, s>>>(bsum, nb);
    us_write_kernel<V, E><<<grid, US_T, 0, s>>>(val, endv, n, nb, bsum, out, end);
    count_launch(3);
}

// 9-significant-digit decimals (the trace format's on-disk precision,
// trace_model.py:63-65): code = m | j << 30, value = m * 10^-(p0 + j) as ONE
// correctly rounded IEEE operation -- the same double a decimal parse of
// "m e-(p0+j)" yields, so the decode is exact.
__constant__ double POW10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                                 1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};

__global__ void dict_bits_decode_kernel(const uint64_t *dict, const uint32_t *w, int width, int64_t n,
                                        uint64_t *out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const uint64_t mask = (1ULL << width) - 1ULL;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const int64_t bit = i * (int64_t)width;
        const int64_t k = bit >> 5;
        const uint64_t win = (uint64_t)__ldg(w + k) | ((uint64_t)__ldg(w + k + 1) << 32);
        __stcs(out + i, __ldg(dict + ((win >> (bit & 31)) & mask)));
    }
}

// Timestamps of a clock with a nominal period, as residuals from the linear
// predictor pred(i) = base + i * step_hi + ((i * step_lo) >> 32) (step =
// step_hi + step_lo / 2^32 us per sample, fixed point): out[i] = pred(i) +
// bias + field i.  A map, not a scan: every element decodes on its own.
__global__ void grid_decode_kernel(const uint32_t *w, int width, int64_t bias, int64_t n, int64_t base,
                                   uint64_t step_hi, uint64_t step_lo, int64_t *out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const uint64_t mask = (1ULL << width) - 1ULL;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const int64_t bit = i * (int64_t)width;
        const int64_t k = bit >> 5;
        const uint64_t win = (uint64_t)__ldg(w + k) | ((uint64_t)__ldg(w + k + 1) << 32);
        const uint64_t pred = (uint64_t)base + (uint64_t)i * step_hi + (((uint64_t)i * step_lo) >> 32);
        __stcs(out + i, (int64_t)(pred + (uint64_t)bias + ((win >> (bit & 31)) & mask)));
    }
}

template <typename T>
__global__ void dict_decode_kernel(const uint64_t *dict, const T *code, int64_t n, uint64_t *out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        __stcs(out + i, __ldg(dict + __ldcs(code + i)));
}

// correctly rounded 1/10^p: with Markstein's final FMA step the quotient
// m / 10^p equals IEEE division for every m < 2^30 and p <= 22 (exhaustive:
// scripts/micro/dec_check.cu, 0 mismatches over 23 x 2^30), at a fraction of
// __ddiv_rn's instructions.
__constant__ double RCP10[23] = {1.0, 0.1, 0.01, 0.001, 0.0001, 1e-05, 1e-06, 1e-07, 1e-08, 1e-09, 1e-10, 1e-11, 1e-12, 1e-13, 1e-14, 1e-15, 1e-16, 1e-17, 1e-18, 1e-19, 1e-20, 1e-21, 1e-22};

__device__ __forceinline__ double decimal_value(uint32_t c, int32_t p0) {
    const double m = (double)(c & 0x3FFFFFFFu);
    const int p = p0 + (int)(c >> 30);
    if (p >= 0) {
        const double y = RCP10[p], d = POW10[p];
        const double q = __dmul_rn(m, y);
        return __fma_rn(__fma_rn(-q, d, m), y, q);
    }
    return __dmul_rn(m, POW10[-p]);
}

__global__ void decimal_decode_kernel(const uint32_t *code, int64_t n, int32_t p0, double *out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        __stcs(out + i, decimal_value(__ldcs(code + i), p0));
}

// ---- run-coded watts: a bitmap marks the samples that carry a new code (bit
// i of word i / 32; sample 0 always does), the codes of those samples only.
// Sample s takes code[popcount of the bitmap over [0, s]] - 1].  Three
// passes: new codes per block of REP_WORDS words, their exclusive scan (one
// block), then the decode: each warp takes 32 words (1024 samples) and writes
// 32 coalesced rows of 32 samples.
constexpr int REP_WORDS = 1024;  // bitmap words per block (32768 samples)

__global__ void __launch_bounds__(256) rep_count_kernel(const uint32_t *rep, int64_t nwords,
                                                        unsigned long long *bsum) {
    __shared__ unsigned ws[8];
    const int64_t w0 = blockIdx.x * (int64_t)REP_WORDS;
    unsigned c = 0;
    for (int k = threadIdx.x; k < REP_WORDS; k += 256)
        if (w0 + k < nwords) c += __popc(__ldg(rep + w0 + k));
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < 8; ++w) t += ws[w];
        bsum[blockIdx.x] = t;
    }
}

// exclusive scan of nb block counts, in place (one block of 1024 threads, 8
// consecutive counts per thread per round)
__global__ void __launch_bounds__(1024) rep_scan_kernel(unsigned long long *bsum, int64_t nb) {
    constexpr int PER = 8, ROUND = 1024 * PER;
    __shared__ unsigned long long wt[32];
    __shared__ unsigned long long carry;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < nb; c0 += ROUND) {
        const int64_t i = c0 + (int64_t)threadIdx.x * PER;
        unsigned long long v[PER], t = 0;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            v[j] = i + j < nb ? bsum[i + j] : 0;
            t += v[j];
        }
        unsigned long long x = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wt[warp] = x;
        __syncthreads();
        unsigned long long off = carry + x - t;
        for (int w = 0; w < warp; ++w) off += wt[w];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            if (i + j < nb) bsum[i + j] = off;
            off += v[j];
        }
        __syncthreads();
        if (threadIdx.x == 1023) carry = off;
        __syncthreads();
    }
}

// the run-coded column's k-th stored code: u32 codes, or bias + the width-bit
// field k (dw_unpack_bits layout)
struct U32Codes {
    const uint32_t *c;
    __device__ __forceinline__ uint32_t operator()(int64_t k) const { return __ldg(c + k); }
};
struct BitCodes {
    const uint32_t *w;
    int width;
    uint32_t bias;
    __device__ __forceinline__ uint32_t operator()(int64_t k) const {
        const int64_t bit = k * (int64_t)width;
        const int64_t q = bit >> 5;
        const uint64_t win = (uint64_t)__ldg(w + q) | ((uint64_t)__ldg(w + q + 1) << 32);
        return bias + (uint32_t)((win >> (bit & 31)) & ((1ULL << width) - 1ULL));
    }
};

template <typename Codes>
__global__ void __launch_bounds__(1024) rep_decode_kernel(Codes code, const uint32_t *rep, int64_t n,
                                                          int32_t p0, const unsigned long long *bpre,
                                                          double *out) {
    __shared__ unsigned wt[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t nwords = (n + 31) >> 5;
    const int64_t wfirst = blockIdx.x * (int64_t)REP_WORDS + warp * 32;  // this warp's first word
    const uint32_t word = wfirst + lane < nwords ? __ldcs(rep + wfirst + lane) : 0u;
    const unsigned pc = __popc(word);
    unsigned inc = pc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) wt[warp] = inc;
    __syncthreads();
    const unsigned off = __reduce_add_sync(0xffffffffu, lane < warp ? wt[lane] : 0u);
    const int64_t base = (int64_t)bpre[blockIdx.x] + off - 1;  // new codes before this warp, minus one
    const unsigned exc = inc - pc;
    const uint32_t upto = 0xFFFFFFFFu >> (31 - lane);  // bits 0 .. lane
#pragma unroll 4
    for (int k = 0; k < 32; ++k) {
        const uint32_t wk = __shfl_sync(0xffffffffu, word, k);
        const unsigned ek = __shfl_sync(0xffffffffu, exc, k);
        const int64_t smp = ((wfirst + k) << 5) + lane;
        if (smp < n) {
            int64_t idx = base + ek + __popc(wk & upto);
            idx = idx < 0 ? 0 : idx;  // only a bitmap without bit 0 (invalid input)
            __stcs(out + smp, decimal_value(code(idx), p0));
        }
    }
}

template <typename Codes>
static int unpack_decimal_rep(Codes codes, const uint32_t *d_rep, int64_t n, int32_t p0, double *d_out,
                              void *d_workspace, size_t workspace_bytes, cudaStream_t s) {
    if (!d_workspace || workspace_bytes < dw_unpack_decimal_rep_workspace_size(n)) return DW_E_WORKSPACE;
    const int64_t nwords = (n + 31) >> 5, nb = ceil_div(nwords, REP_WORDS);
    unsigned long long *bsum = (unsigned long long *)d_workspace;
    rep_count_kernel<<<(unsigned)nb, 256, 0, s>>>(d_rep, nwords, bsum);
    rep_scan_kernel<<<1, 1024, 0, s>>>(bsum, nb);
    rep_decode_kernel<<<(unsigned)nb, 1024, 0, s>>>(codes, d_rep, n, p0, bsum, d_out);
    count_launch(3);
    DW_CHECK_LAUNCH();
    return DW_OK;
}

}  // namespace dw

using namespace dw;

extern "C" {

size_t dw_unpack_workspace_size(int64_t n) { return 8 * (size_t)(ceil_div(std::max<int64_t>(n, 1), US_B) + 1) + 256; }

int dw_unpack_deltas_w(const void *d_delta, int32_t delta_bytes, int64_t delta_bias, int64_t n, int64_t base,
                       int64_t *d_out, const void *d_dur, int32_t dur_bytes, int64_t *d_end, void *d_workspace,
                       size_t workspace_bytes, dw_stream_t stream) {
    if (n < 0 || (n && (!d_delta || !d_out)) || (d_dur && !d_end) || n >= ((int64_t)1 << 31)) return DW_E_ARG;
    if ((delta_bytes != 1 && delta_bytes != 2 && delta_bytes != 4) ||
        (d_dur && dur_bytes != 2 && dur_bytes != 4))
        return DW_E_ARG;
    if (n == 0) return DW_OK;
    if (!d_workspace || workspace_bytes < dw_unpack_workspace_size(n)) return DW_E_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    auto go = [&](auto val) {
        if (!d_dur) unpack_scan(val, NoEnd{}, n, d_out, nullptr, d_workspace, s);
        else if (dur_bytes == 2) unpack_scan(val, DurAt<uint16_t>{(const uint16_t *)d_dur}, n, d_out, d_end, d_workspace, s);
        else unpack_scan(val, DurAt<uint32_t>{(const uint32_t *)d_dur}, n, d_out, d_end, d_workspace, s);
    };
    if (delta_bytes == 1) go(DeltaAt<int8_t>{(const int8_t *)d_delta, base, delta_bias});
    else if (delta_bytes == 2) go(DeltaAt<uint16_t>{(const uint16_t *)d_delta, base, delta_bias});
    else go(DeltaAt<uint32_t>{(const uint32_t *)d_delta, base, delta_bias});
    DW_CHECK_LAUNCH();
    return DW_OK;
}

int dw_unpack_bits(const uint32_t *d_words, int32_t width, int64_t bias, int64_t n, int64_t base, int64_t *d_out,
                   void *d_workspace, size_t workspace_bytes, dw_stream_t stream) {
    if (n < 0 || width < 1 || width > 32 || (n && (!d_words || !d_out)) || n >= ((int64_t)1 << 31)) return DW_E_ARG;
    if (n == 0) return DW_OK;
    if (!d_workspace || workspace_bytes < dw_unpack_workspace_size(n)) return DW_E_WORKSPACE;
    unpack_scan(BitsAt{d_words, width, base, bias}, NoEnd{}, n, d_out, nullptr, d_workspace, (cudaStream_t)stream);
    DW_CHECK_LAUNCH();
    return DW_OK;
}

int dw_unpack_bits_w(const uint32_t *d_words, int32_t width, int64_t bias, int64_t n, int64_t base, int64_t *d_out,
                     const uint32_t *d_dur_words, int32_t dur_width, int64_t dur_bias, int64_t *d_end,
                     void *d_workspace, size_t workspace_bytes, dw_stream_t stream) {
    if (!d_dur_words)
        return dw_unpack_bits(d_words, width, bias, n, base, d_out, d_workspace, workspace_bytes, stream);
    if (n < 0 || width < 1 || width > 32 || dur_width < 1 || dur_width > 32 || (n && (!d_words || !d_out || !d_end)) ||
        n >= ((int64_t)1 << 31))
        return DW_E_ARG;
    if (n == 0) return DW_OK;
    if (!d_workspace || workspace_bytes < dw_unpack_workspace_size(n)) return DW_E_WORKSPACE;
    unpack_scan(BitsAt{d_words, width, base, bias}, BitsDurAt{d_dur_words, dur_width, dur_bias}, n, d_out, d_end,
                d_workspace, (cudaStream_t)stream);
    DW_CHECK_LAUNCH();
    return DW_OK;
}

int dw_unpack_bits_dur(const int64_t *d_start, const uint32_t *d_words, int32_t width, int64_t bias, int64_t n,
                       int64_t *d_end, dw_stream_t stream) {
    if (n < 0 || width < 1 || width > 32 || (n && (!d_start || !d_words || !d_end))) return DW_E_ARG;
    if (n) {
        add_bits_duration_kernel<<<(unsigned)std::min<int64_t>(num_sms() * 8, ceil_div(n, 256)), 256, 0,
                                   (cudaStream_t)stream>>>(d_start, d_words, width, bias, n, d_end);
        count_launch();
    }
    DW_CHECK_LAUNCH();
    return DW_OK;
}

int dw_unpack_grid(const uint32_t *d_words, int32_t width, int64_t bias, int64_t n, int64_t base, uint64_t step_fx,
                   int64_t *d_out, dw_stream_t stream) {
    // i * step_lo < 2^63 and i * step_hi < 2^63 need n < 2^31 and step_hi < 2^31
    if (n < 0 || width < 1 || width > 32 || (n && (!d_words || !d_out)) || n >= ((int64_t)1 << 31) ||
        (step_fx >> 63))
        return DW_E_ARG;
    if (n) {
        grid_decode_kernel<<<(unsigned)std::min<int64_t>(num_sms() * 8, ceil_div(n, 256)), 256, 0,
                             (cudaStream_t)stream>>>(d_words, width, bias, n, base, step_fx >> 32,
                                                     step_fx & 0xFFFFFFFFULL, d_out);
        count_launch();
    }
    DW_CHECK_LAUNCH();
    return DW_OK;
}

int dw_unpack_dict_bits(const uint64_t *d_dict, const uint32_t *d_words, int32_t width, int64_t n, uint64_t *d_out,
                        dw_stream_t stream) {
    if (n < 0 || width < 1 || width > 32 || (n && (!d_dict || !d_words || !d_out))) return DW_E_ARG;
    if (n) {
        dict_bits_decode_kernel<<<(unsigned)std::min<int64_t>(num_sms() * 8, ceil_div(n, 256)), 256, 0,
                                  (cudaStream_t)stream>>>(d_dict, d_words, width, n, d_out);
        count_launch();
    }
    DW_CHECK_LAUNCH();
    return DW_OK;
}

int dw_unpack_dict(const uint64_t *d_dict, const void *d_code, int32_t code_bytes, int64_t n, uint64_t *d_out,
                   dw_stream_t stream) {
    if (n < 0 || (n && (!d_dict || !d_code || !d_out)) || (code_bytes != 2 && code_bytes != 4)) return DW_E_ARG;
    if (n) {
        const unsigned grid = (unsigned)std::min<int64_t>(num_sms() * 8, ceil_div(n, 256));
        if (code_bytes == 2)
            dict_decode_kernel<uint16_t><<<grid, 256, 0, (cudaStream_t)stream>>>(d_dict, (const uint16_t *)d_code,
                                                                                 n, d_out);
        else
            dict_decode_kernel<uint32_t><<<grid, 256, 0, (cudaStream_t)stream>>>(d_dict, (const uint32_t *)d_code,
                                                                                 n, d_out);
        count_launch();
    }
    DW_CHECK_LAUNCH();
    return DW_OK;
}

int dw_unpack_deltas(const uint32_t *d_delta, int64_t n, int64_t base, int64_t *d_out, const uint32_t *d_dur,
                     int64_t *d_end, void *d_workspace, size_t workspace_bytes, dw_stream_t stream) {
    return dw_unpack_deltas_w(d_delta, 4, 0, n, base, d_out, d_dur, 4, d_end, d_workspace, workspace_bytes, stream);
}

size_t dw_unpack_decimal_rep_workspace_size(int64_t n) {
    const int64_t nwords = (std::max<int64_t>(n, 0) + 31) >> 5;
    return 8 * (size_t)(ceil_div(nwords, REP_WORDS) + 1) + 256;
}

int dw_unpack_decimal_rep(const uint32_t *d_code, const uint32_t *d_rep, int64_t n, int32_t p0, double *d_out,
                          void *d_workspace, size_t workspace_bytes, dw_stream_t stream) {
    if (n < 0 || (n && (!d_code || !d_rep || !d_out)) || p0 < -22 || p0 + 3 > 22) return DW_E_ARG;
    if (n == 0) return DW_OK;
    return unpack_decimal_rep(U32Codes{d_code}, d_rep, n, p0, d_out, d_workspace, workspace_bytes,
                              (cudaStream_t)stream);
}

int dw_unpack_decimal_rep_bits(const uint32_t *d_words, int32_t width, uint32_t bias, const uint32_t *d_rep, int64_t n,
                               int32_t p0, double *d_out, void *d_workspace, size_t workspace_bytes,
                               dw_stream_t stream) {
    if (n < 0 || width < 1 || width > 32 || (n && (!d_words || !d_rep || !d_out)) || p0 < -22 || p0 + 3 > 22)
        return DW_E_ARG;
    if (n == 0) return DW_OK;
    return unpack_decimal_rep(BitCodes{d_words, width, bias}, d_rep, n, p0, d_out, d_workspace, workspace_bytes,
                              (cudaStream_t)stream);
}

int dw_unpack_decimal(const uint32_t *d_code, int64_t n, int32_t p0, double *d_out, dw_stream_t stream) {
    if (n < 0 || (n && (!d_code || !d_out)) || p0 < -22 || p0 + 3 > 22) return DW_E_ARG;
    if (n) {
        decimal_decode_kernel<<<(unsigned)std::min<int64_t>(num_sms() * 8, ceil_div(n, 256)), 256, 0,
                                (cudaStream_t)stream>>>(d_code, n, p0, d_out);
        count_launch();
    }
    DW_CHECK_LAUNCH();
    return DW_OK;
}

}  // extern "C"
