// split.cu -- overlap-split attribution (G1) on B200 (sm_100a).
//
// The reference gives every interval the full signal energy over its span, so
// concurrent kernels double-count (energy.py:305-316 integrates
// each interval independently).  This mode divides the power equally among
// the intervals of one set that are active at each instant (DESIGN.md
// "overlap split"; CPU restatement: oracle/dw_oracle.c dwo_split):
//
//   x_0 < ... < x_{u-1}  distinct endpoints of the set's non-empty intervals
//   slice k = [x_k, x_{k+1}],  c_k = intervals active over the whole slice
//   e_k     = compat integral of the slice (dw_attribute: bit-identical to the
//             reference's sequential sum up to DW_DIRECT_MAX segments)
//   share_k = e_k / c_k (0 if c_k == 0)
//   joules  = share_k for a one-slice interval, else the exact (2^-64 J fixed
//             point) sum of its slices' shares rounded once; 0 if empty.
//
// Without overlap every interval is a single slice with c = 1, so the result
// equals the compat path bit for bit.  Device steps: endpoint events ->
// radix sort by time -> inclusive scan of +1/-1 (active counts) -> run ids ->
// slice integrals through the tile kernel -> int128 exclusive scan of the
// fixed-point shares -> one difference per interval.  Sort and scan traffic
// is implementation overhead.
#include <algorithm>

#include <cub/cub.cuh>

#include "dw_common.cuh"

namespace dw {

struct U128 {
    unsigned long long lo, hi;
};
struct U128Sum {
    __device__ __forceinline__ U128 operator()(const U128 &a, const U128 &b) const {
        U128 r;
        r.lo = a.lo + b.lo;
        r.hi = a.hi + b.hi + (r.lo < a.lo);
        return r;
    }
};

constexpr int SP_THREADS = 256;

// events: start of interval k at 2k, end at 2k+1; empty intervals get the
// sentinel key (sorted last).  Keys are times relative to the span start.
__global__ void split_events_kernel(const int64_t *lo, const int64_t *hi, int64_t n, int64_t t0,
                                    int64_t span_lo, int64_t span_hi, uint64_t sentinel,
                                    uint64_t *key, uint32_t *val, unsigned long long *bad,
                                    unsigned long long *n_events) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    unsigned c = 0;
    if (k < n) {
        const int64_t a = lo[k], b = hi[k];
        if (b < a || a < span_lo || b > span_hi) atomicMin(bad, (unsigned long long)k);
        const bool live = b > a;
        key[2 * k] = live ? (uint64_t)(a - t0) : sentinel;
        key[2 * k + 1] = live ? (uint64_t)(b - t0) : sentinel;
        val[2 * k] = (uint32_t)(2 * k);
        val[2 * k + 1] = (uint32_t)(2 * k + 1);
        c = live ? 2u : 0u;
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(n_events, (unsigned long long)c);
}

// +1 for a start, -1 for an end; run-start flags of equal keys
__global__ void split_tags_kernel(const uint64_t *key, const uint32_t *val, int64_t ne, int32_t *tag,
                                  int32_t *first) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= ne) return;
    tag[e] = (val[e] & 1u) ? -1 : 1;
    first[e] = (e == 0 || key[e] != key[e - 1]) ? 1 : 0;
}

// per event: its run id (= slice index of its time); per run end: x, c
__global__ void split_runs_kernel(const uint64_t *key, const uint32_t *val, int64_t ne, int64_t t0,
                                  const int32_t *active, const int32_t *run_incl, int64_t *x,
                                  int32_t *c, int32_t *slice_of_ev) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= ne) return;
    const int32_t r = run_incl[e] - 1;
    slice_of_ev[val[e]] = r;
    if (e == ne - 1 || key[e + 1] != key[e]) {
        x[r] = (int64_t)key[e] + t0;
        c[r] = active[e];
    }
}

// slice ends (a separate 16-byte aligned column for the tile kernel's bulk copies)
__global__ void split_slice_end_kernel(const int64_t *x, int64_t ns, int64_t *xe) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < ns) xe[k] = x[k + 1];
}

__global__ void split_shares_kernel(double *es, const int32_t *c, int64_t ns, U128 *q) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= ns) return;
    const double sh = c[k] > 0 ? __ddiv_rn(es[k], (double)c[k]) : 0.0;
    es[k] = sh;
    const I128Parts pp = split(fx_from_double(sh, FX_JOULE_BITS));
    q[k] = U128{pp.lo, pp.hi};
}

__global__ void split_prefix_end_kernel(const U128 *q, U128 *P, int64_t ns) {
    if (threadIdx.x == 0) P[ns] = U128Sum()(P[ns - 1], q[ns - 1]);
}

__global__ void split_final_kernel(const int64_t *lo, const int64_t *hi, int64_t n, const int32_t *slice_of_ev,
                                   const double *share, const U128 *P, double *out) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    if (hi[k] <= lo[k]) {  // empty (or invalid: reported through the status block)
        out[k] = 0.0;
        return;
    }
    const int32_t a = slice_of_ev[2 * k], b = slice_of_ev[2 * k + 1];
    if (b == a + 1) {
        out[k] = share[a];
    } else {
        const i128 d = join(P[b].lo, P[b].hi) - join(P[a].lo, P[a].hi);
        out[k] = fx_to_double(d, FX_JOULE_BITS);
    }
}

__global__ void split_report_kernel(DevStatus *st, const unsigned long long *bad) {
    if (threadIdx.x == 0 && *bad != (unsigned long long)NONE) atomicMin(&st->bad_index[0], *bad);
}

static size_t au(size_t x) { return (x + 255) & ~(size_t)255; }

struct SplitLayout {
    size_t attr, counters, key, key2, val, val2, tag, first, active, run, x, xe, c, ev_slice, es, q, P,
        cub, cub_bytes, total;
};

static SplitLayout split_layout(int64_t S, int64_t n) {
    SplitLayout L{};
    const int64_t ne = 2 * std::max<int64_t>(n, 1);
    const int64_t ns = ne;  // slices <= distinct endpoints
    size_t off = 0;
    const int64_t sizes[1] = {ns};
    L.attr = off; off += au(dw_attribute_workspace_size(S, sizes, 1));
    L.counters = off; off += au(64);
    L.key = off; off += au(8 * ne);
    L.key2 = off; off += au(8 * ne);
    L.val = off; off += au(4 * ne);
    L.val2 = off; off += au(4 * ne);
    L.tag = off; off += au(4 * ne);
    L.first = off; off += au(4 * ne);
    L.active = off; off += au(4 * ne);
    L.run = off; off += au(4 * ne);
    L.x = off; off += au(8 * (ns + 1));
    L.xe = off; off += au(8 * (ns + 1));
    L.c = off; off += au(4 * (ns + 1));
    L.ev_slice = off; off += au(4 * ne);
    L.es = off; off += au(8 * (ns + 1));
    L.q = off; off += au(16 * (ns + 1));
    L.P = off; off += au(16 * (ns + 2));
    size_t c1 = 0, c2 = 0, c3 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, c1, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                    (const uint32_t *)nullptr, (uint32_t *)nullptr, (int)ne);
    cub::DeviceScan::InclusiveSum(nullptr, c2, (const int32_t *)nullptr, (int32_t *)nullptr, (int)ne);
    cub::DeviceScan::ExclusiveScan(nullptr, c3, (const U128 *)nullptr, (U128 *)nullptr, U128Sum(), U128{0, 0},
                                   (int)(ns + 1));
    L.cub = off;
    L.cub_bytes = std::max(c1, std::max(c2, c3));
    off += au(L.cub_bytes);
    L.total = off;
    return L;
}

static int bits_for_u64(uint64_t v) {
    int b = 1;
    while (b < 64 && (v >> b)) ++b;
    return b;
}

}  // namespace dw

using namespace dw;

extern "C" {

size_t dw_attribute_split_workspace_size(int64_t n_samples, int64_t n) {
    return split_layout(n_samples, n).total;
}

int dw_attribute_split(const dw_signal_t *sig, dw_interval_set_t *set, void *d_workspace, size_t workspace_bytes,
                       dw_stream_t stream) {
    if (!sig || !set || !d_workspace || set->n < 0) return DW_E_ARG;
    if (sig->kind != DW_SIGNAL_STEP && sig->kind != DW_SIGNAL_LINEAR) return DW_E_ARG;
    const int64_t n = set->n, S = sig->n;
    if (n > ((int64_t)1 << 30)) return DW_E_ARG;  // event ids are 32-bit
    if (n && (!set->d_start || !set->d_end || !set->d_joules)) return DW_E_ARG;
    SplitLayout L = split_layout(S, n);
    if (workspace_bytes < L.total) return DW_E_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    char *base = (char *)d_workspace;
    if (S <= 0 || !sig->d_ts || !sig->d_watts) {
        dw_interval_set_t none{};
        return dw_attribute(sig, &none, 0, base + L.attr, L.counters - L.attr, stream);  // DW_E_EMPTY
    }
    // span of the signal (host needs it for the sort's key width)
    int64_t t_first = 0, t_last = 0;
    cudaMemcpyAsync(&t_first, sig->d_ts, 8, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&t_last, sig->d_ts + S - 1, 8, cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return DW_E_CUDA;
    const int64_t span_hi = sig->kind == DW_SIGNAL_STEP ? sig->span_hi : t_last;
    const uint64_t range = (uint64_t)(span_hi > t_first ? span_hi - t_first : 0);
    const uint64_t sentinel = range + 1;
    const int end_bit = bits_for_u64(sentinel);

    unsigned long long *ctr = (unsigned long long *)(base + L.counters);  // [0] bad, [1] events
    uint64_t *key = (uint64_t *)(base + L.key), *key2 = (uint64_t *)(base + L.key2);
    uint32_t *val = (uint32_t *)(base + L.val), *val2 = (uint32_t *)(base + L.val2);
    int32_t *tag = (int32_t *)(base + L.tag), *first = (int32_t *)(base + L.first);
    int32_t *active = (int32_t *)(base + L.active), *run = (int32_t *)(base + L.run);
    int64_t *x = (int64_t *)(base + L.x), *xe = (int64_t *)(base + L.xe);
    int32_t *c = (int32_t *)(base + L.c), *ev_slice = (int32_t *)(base + L.ev_slice);
    double *es = (double *)(base + L.es);
    U128 *q = (U128 *)(base + L.q), *P = (U128 *)(base + L.P);

    const unsigned long long init[2] = {(unsigned long long)NONE, 0ULL};
    cudaMemcpyAsync(ctr, init, sizeof(init), cudaMemcpyHostToDevice, s);
    int64_t ne = 0;
    if (n) {
        const unsigned g = (unsigned)ceil_div(n, SP_THREADS);
        split_events_kernel<<<g, SP_THREADS, 0, s>>>(set->d_start, set->d_end, n, t_first, t_first, span_hi,
                                                    sentinel, key, val, ctr, ctr + 1);
        count_launch();
        size_t cb = L.cub_bytes;
        cub::DeviceRadixSort::SortPairs(base + L.cub, cb, key, key2, val, val2, (int)(2 * n), 0, end_bit, s);
        count_launch(4);
        unsigned long long h[2];
        cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) return DW_E_CUDA;
        ne = (int64_t)h[1];
    }
    int64_t u = 0;
    if (ne) {
        const unsigned g = (unsigned)ceil_div(ne, SP_THREADS);
        split_tags_kernel<<<g, SP_THREADS, 0, s>>>(key2, val2, ne, tag, first);
        size_t cb = L.cub_bytes;
        cub::DeviceScan::InclusiveSum(base + L.cub, cb, tag, active, (int)ne, s);
        cb = L.cub_bytes;
        cub::DeviceScan::InclusiveSum(base + L.cub, cb, first, run, (int)ne, s);
        split_runs_kernel<<<g, SP_THREADS, 0, s>>>(key2, val2, ne, t_first, active, run, x, c, ev_slice);
        count_launch(4);
        int32_t ru = 0;
        cudaMemcpyAsync(&ru, run + ne - 1, 4, cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) return DW_E_CUDA;
        u = ru;
    }
    const int64_t ns = u > 1 ? u - 1 : 0;
    // slice integrals through the compat tile kernel (its status block heads the workspace)
    int rc;
    {
        if (ns) {
            split_slice_end_kernel<<<(unsigned)ceil_div(ns, SP_THREADS), SP_THREADS, 0, s>>>(x, ns, xe);
            count_launch();
        }
        dw_interval_set_t slices{};
        slices.d_start = x;
        slices.d_end = xe;
        slices.n = ns;
        slices.d_joules = es;
        slices.sorted = 1;
        dw_signal_t sg = *sig;
        sg.validate_order = sig->validate_order;
        rc = dw_attribute(&sg, &slices, 1, base + L.attr, L.counters - L.attr, stream);
        if (rc != DW_OK) return rc;
    }
    if (ns) {
        const unsigned g = (unsigned)ceil_div(ns, SP_THREADS);
        split_shares_kernel<<<g, SP_THREADS, 0, s>>>(es, c, ns, q);
        size_t cb = L.cub_bytes;
        cub::DeviceScan::ExclusiveScan(base + L.cub, cb, q, P, U128Sum(), U128{0, 0}, (int)ns, s);
        count_launch(2);
        split_prefix_end_kernel<<<1, 32, 0, s>>>(q, P, ns);  // P[ns]: the end of the last slice
        count_launch();
    }
    if (n) {
        split_final_kernel<<<(unsigned)ceil_div(n, SP_THREADS), SP_THREADS, 0, s>>>(
            set->d_start, set->d_end, n, ev_slice, es, P, set->d_joules);
        count_launch();
    }
    split_report_kernel<<<1, 32, 0, s>>>((DevStatus *)(base + L.attr), ctr);
    count_launch();
    DW_CHECK_LAUNCH();
    return DW_OK;
}

}  // extern "C"
