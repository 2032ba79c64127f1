// attribute.cu -- per-interval energy attribution on B200 (sm_100a).
//
// Replaces the hot loop of the reference's build_ledger: one energy.integrate
// call per operator and per kernel (energy.py:305-316), each an O(S) scan over
// every power segment (energy.py:99-104) or, for a sampled view, a trapezoid
// over rebuilt sample lists (energy.py:108-130).
//
// Data layout (SoA in HBM):
//   power   ts int64[S] (strictly increasing), watts f64[S]
//   sets    start int64[n], end int64[n] (sorted by start), joules f64[n] out
//
// Kernels, in launch order:
//   K0 status_init        reset the status block in the workspace
//   (sort)                only for sets given unsorted: CUB radix sort of start
//   K1 partition          first[set][tile] = first interval whose start >= ts[tile*T]
//   K2 attribute_tiles    persistent CTAs walk sample tiles of T segments.  Each
//                         tile window (T + DIRECT_MAX + 2 samples) is staged in
//                         shared memory by 1-D TMA (cp.async.bulk + mbarrier),
//                         double buffered.  Per tile the CTA (a) checks power
//                         timestamps are strictly increasing, (b) sums the tile's
//                         integrand terms exactly in int128 fixed point (the
//                         "tile prefix" level), (c) integrates every interval whose
//                         start falls in the tile: a shared-memory binary search for
//                         the first segment, then the reference's sequential fp64
//                         sum (bit-identical) for <= DIRECT_MAX segments; longer
//                         intervals go to a list for K4.
//   K3 tile_scan          exclusive scan of the int128 tile sums
//   K4 long_intervals     one warp per long interval: exact fixed-point sum of
//                         partial first/last tiles + prefix difference
//   K5 fx_sum / finalize  operator_total (exact sum) and total / idle
#include <algorithm>

#include <cub/cub.cuh>

#include "dw_common.cuh"

namespace dw {

constexpr int TILE = 2048;                   // segments per tile
constexpr int DIRECT = DW_DIRECT_MAX;        // sequential-sum cap
constexpr int WIN = TILE + DIRECT + 6;       // window slots: 2 halo + TILE + DIRECT + 2, + virtual end
constexpr int ATTR_THREADS = 256;
constexpr int ATTR_WARPS = ATTR_THREADS / 32;

struct AttrParams {
    const int64_t *ts;
    const double *w;
    int64_t S;
    int64_t span_hi;  // step: end of the last segment
    int64_t ntiles;
    int32_t kind;
    int32_t nsets;
    int32_t validate_order;
    int32_t pad;
    const int64_t *start[DW_MAX_SETS];
    const int64_t *end[DW_MAX_SETS];
    double *out[DW_MAX_SETS];
    const int64_t *perm[DW_MAX_SETS];  // sorted position -> caller index (unsorted sets)
    int64_t n[DW_MAX_SETS];
    int32_t check_sorted[DW_MAX_SETS];
    const int64_t *first;        // [nsets][ntiles + 1]
    unsigned long long *tile_fx; // [ntiles][2] (lo, hi)
    unsigned long long *prefix;  // [ntiles + 1][2]
    unsigned long long *long_list;
    DevStatus *st;
};

// ---------------------------------------------------------------- integrands
// Segment i of a step signal: [ts[i], ts[i+1]) (last one ends at span_hi),
// term = w[i] * width.  Piece j of a sampled signal: [ts[j], ts[j+1]],
// term = 0.5 * (v(ts[j]) + v(ts[j+1])) * width with v() of energy.py:115-124.

// v(ts[j]) for a sample time (energy.py:115-124: t <= ts[0] -> ws[0];
// t >= ts[-1] -> ws[-1]; else the FIRST bracketing pair, which for an interior
// sample is (j-1, j) with frac == 1.0).
template <typename TsF, typename WF>
__device__ __forceinline__ double lin_sample_value(int64_t j, int64_t S, TsF ts, WF w) {
    if (j == 0) return w(0);
    if (j == S - 1) return w(S - 1);
    double wa = w(j - 1);
    double frac = __ddiv_rn((double)(ts(j) - ts(j - 1)), (double)(ts(j) - ts(j - 1)));
    return __dadd_rn(wa, __dmul_rn(frac, __dsub_rn(w(j), wa)));
}

// v(t) for an arbitrary time inside the span; lbj = first index with ts >= t.
// (ts0, tsl, w0, wl) are the signal's first/last sample, passed explicitly so
// the accessors only ever touch the neighbourhood of t.
template <typename TsF, typename WF>
__device__ __forceinline__ double lin_value_at(int64_t t, int64_t lbj, int64_t ts0, int64_t tsl,
                                               double w0, double wl, TsF ts, WF w) {
    if (t <= ts0) return w0;
    if (t >= tsl) return wl;
    int64_t i = lbj - 1;
    double wa = w(i);
    double frac = __ddiv_rn((double)(t - ts(i)), (double)(ts(i + 1) - ts(i)));
    return __dadd_rn(wa, __dmul_rn(frac, __dsub_rn(w(i + 1), wa)));
}

__device__ __forceinline__ double lin_piece(double va, double vb, int64_t width) {
    return __dmul_rn(__dmul_rn(0.5, __dadd_rn(va, vb)), (double)width);
}

// --------------------------------------------------------------- K0 status
__global__ void status_init_kernel(DevStatus *st) {
    int t = threadIdx.x;
    if (t < DW_MAX_SETS) {
        st->bad_index[t] = (unsigned long long)NONE;
        st->unsorted_index[t] = (unsigned long long)NONE;
    }
    if (t == 0) {
        st->order_index = (unsigned long long)NONE;
        st->long_count = 0;
    }
    if (t < 4) st->totals[t] = 0.0;
}

// ------------------------------------------------------------ K1 partition
__global__ void partition_kernel(AttrParams p) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t nb = p.ntiles + 1;
    if (b >= nb * p.nsets) return;
    int j = (int)(b / nb);
    b -= (int64_t)j * nb;
    int64_t n = p.n[j];
    int64_t r;
    if (b == 0) {
        r = 0;
    } else if (b == p.ntiles) {
        r = n;
    } else {
        int64_t key = p.ts[b * TILE];
        const int64_t *a = p.start[j];
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            int64_t mid = lo + ((hi - lo) >> 1);
            if (__ldg(a + mid) < key) lo = mid + 1; else hi = mid;
        }
        r = lo;
    }
    const_cast<int64_t *>(p.first)[j * nb + b] = r;
}

// --------------------------------------------------------- K2 tile kernel
struct __align__(16) TileSmem {
    int64_t ts[2][WIN];
    double w[2][WIN];
    uint64_t bar[2];
    unsigned long long red[ATTR_WARPS][2];
    int64_t win_base[2];
    int64_t win_cnt[2];
};

__device__ __forceinline__ void tile_window(int64_t tile, int64_t S, int64_t &wb, int64_t &we) {
    wb = tile * TILE - 2;
    if (wb < 0) wb = 0;
    we = (tile + 1) * TILE + DIRECT + 2;  // keeps the steady-state window even (16-B TMA)
    if (we > S) we = S;
}

__device__ __forceinline__ void issue_tile(const AttrParams &p, TileSmem &sm, int stage,
                                           int64_t tile) {
    int64_t wb, we;
    tile_window(tile, p.S, wb, we);
    int64_t cnt = we - wb;
    int64_t even = cnt & ~(int64_t)1;
    uint32_t bytes = (uint32_t)(even * 8);
    sm.win_base[stage] = wb;
    sm.win_cnt[stage] = cnt;
    mbar_expect_tx(&sm.bar[stage], 2 * bytes);
    if (bytes) {
        tma_load_1d(sm.ts[stage], p.ts + wb, bytes, &sm.bar[stage]);
        tma_load_1d(sm.w[stage], p.w + wb, bytes, &sm.bar[stage]);
    }
}

__device__ __forceinline__ void report_bad(const AttrParams &p, int j, int64_t k) {
    int64_t idx = p.perm[j] ? __ldg(p.perm[j] + k) : k;
    atomic_min_index(&p.st->bad_index[j], idx);
}

__device__ __forceinline__ void push_long(const AttrParams &p, int j, int64_t k) {
    unsigned long long slot = atomicAdd(&p.st->long_count, 1ULL);
    p.long_list[slot] = ((unsigned long long)j << 56) | (unsigned long long)k;
}

template <int KIND>
__global__ void __launch_bounds__(ATTR_THREADS, 3) attribute_tiles_kernel(AttrParams p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    TileSmem &sm = *reinterpret_cast<TileSmem *>(smem_raw);
    const int tid = threadIdx.x;
    int64_t tile = blockIdx.x;
    if (tile >= p.ntiles) return;

    const int64_t S = p.S;
    const int64_t ts0 = __ldg(p.ts);
    const int64_t tsl = __ldg(p.ts + S - 1);
    const int64_t span_lo = ts0;
    const int64_t span_hi = KIND == DW_SIGNAL_STEP ? p.span_hi : tsl;
    const int64_t nterms = KIND == DW_SIGNAL_STEP ? S : S - 1;
    const double w0 = __ldg(p.w), wl = __ldg(p.w + S - 1);

    if (tid == 0) {
        mbar_init(&sm.bar[0], 1);
        mbar_init(&sm.bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) issue_tile(p, sm, 0, tile);

    for (int it = 0; tile < p.ntiles; tile += gridDim.x, ++it) {
        const int stage = it & 1;
        const int64_t next = tile + gridDim.x;
        if (tid == 0 && next < p.ntiles) {
            fence_proxy_async();
            issue_tile(p, sm, stage ^ 1, next);
        }
        mbar_wait(&sm.bar[stage], (uint32_t)((it >> 1) & 1));
        const int64_t wb = sm.win_base[stage];
        const int64_t cnt = sm.win_cnt[stage];
        int64_t *s_ts = sm.ts[stage];
        double *s_w = sm.w[stage];
        if (tid == 0) {
            if (cnt & 1) {  // odd tail: not a 16-byte multiple, load directly
                s_ts[cnt - 1] = __ldg(p.ts + wb + cnt - 1);
                s_w[cnt - 1] = __ldg(p.w + wb + cnt - 1);
            }
            if (wb + cnt == S) s_ts[cnt] = span_hi;  // virtual end of the last segment
        }
        __syncthreads();

        const int64_t t0 = tile * TILE;                            // first segment of the tile
        const int64_t t1 = min((tile + 1) * TILE, S);              // one past the last sample
        auto TS = [&](int64_t g) -> int64_t { return s_ts[g - wb]; };
        auto W = [&](int64_t g) -> double { return s_w[g - wb]; };

        // (a) strictly increasing timestamps (trace_model.py:549-551)
        if (p.validate_order) {
            for (int64_t i = t0 + tid; i < min(t1, S - 1); i += ATTR_THREADS)
                if (TS(i + 1) <= TS(i)) atomic_min_index(&p.st->order_index, i);
        }

        // (b) exact tile sum of the integrand terms (the tile-prefix level)
        {
            i128 acc = 0;
            const int64_t e1 = min((tile + 1) * TILE, nterms);
            for (int64_t i = t0 + tid; i < e1; i += ATTR_THREADS) {
                double term;
                if (KIND == DW_SIGNAL_STEP) {
                    term = __dmul_rn(W(i), (double)(TS(i + 1) - TS(i)));
                } else {
                    double va = lin_sample_value(i, S, TS, W);
                    double vb = lin_sample_value(i + 1, S, TS, W);
                    term = lin_piece(va, vb, TS(i + 1) - TS(i));
                }
                acc += q_term(term);
            }
            acc = warp_sum_i128(acc);
            if ((tid & 31) == 0) {
                I128Parts pp = split(acc);
                sm.red[tid >> 5][0] = pp.lo;
                sm.red[tid >> 5][1] = pp.hi;
            }
            __syncthreads();
            if (tid == 0) {
                i128 s = 0;
#pragma unroll
                for (int k = 0; k < ATTR_WARPS; ++k) s += join(sm.red[k][0], sm.red[k][1]);
                I128Parts pp = split(s);
                p.tile_fx[2 * tile] = pp.lo;
                p.tile_fx[2 * tile + 1] = pp.hi;
            }
        }

        // (c) intervals whose start falls in this tile
        for (int j = 0; j < p.nsets; ++j) {
            const int64_t f0 = p.first[j * (p.ntiles + 1) + tile];
            const int64_t f1 = p.first[j * (p.ntiles + 1) + tile + 1];
            const int64_t *st_a = p.start[j];
            const int64_t *en_a = p.end[j];
            for (int64_t k = f0 + tid; k < f1; k += ATTR_THREADS) {
                const int64_t lo = __ldg(st_a + k);
                const int64_t hi = __ldg(en_a + k);
                if (p.check_sorted[j] && k > 0 && __ldg(st_a + k - 1) > lo)
                    atomic_min_index(&p.st->unsorted_index[j], k);
                if (hi < lo || lo < span_lo || hi > span_hi) {
                    report_bad(p, j, k);
                    continue;
                }
                const int64_t oidx = p.perm[j] ? __ldg(p.perm[j] + k) : k;
                double tot = 0.0;
                bool is_long = false;
                if (KIND == DW_SIGNAL_STEP) {
                    // last segment start <= lo, searched in [t0, t1)
                    int64_t l = t0, h = t1;  // upper_bound(lo) in [t0, t1)
                    while (l < h) {
                        int64_t m = (l + h) >> 1;
                        if (TS(m) <= lo) l = m + 1; else h = m;
                    }
                    int64_t i = l - 1;
                    if (i < t0) i = t0;
                    int nseg = 0;
                    for (; i < S && TS(i) < hi; ++i) {
                        if (nseg == DIRECT) { is_long = true; break; }
                        int64_t s = TS(i), e = TS(i + 1);
                        int64_t ov = min(e, hi) - max(s, lo);
                        tot = __dadd_rn(tot, __dmul_rn(W(i), (double)ov));
                        ++nseg;
                    }
                } else {
                    // first sample > lo, searched in [t0, t1]
                    int64_t l = t0, h = t1;
                    while (l < h) {
                        int64_t m = (l + h) >> 1;
                        if (TS(m) <= lo) l = m + 1; else h = m;
                    }
                    const int64_t first = l;
                    const int64_t lbj = (first > 0 && TS(first - 1) == lo) ? first - 1 : first;
                    double vprev = lin_value_at(lo, lbj, ts0, tsl, w0, wl, TS, W);
                    int64_t prev = lo;
                    int64_t j2 = first;
                    int m = 0;
                    for (; j2 < S && TS(j2) < hi; ++j2) {
                        // pieces = interior points + 1; more than DIRECT pieces -> long
                        if (m == DIRECT - 1) { is_long = true; break; }
                        double vj = lin_sample_value(j2, S, TS, W);
                        tot = __dadd_rn(tot, lin_piece(vprev, vj, TS(j2) - prev));
                        prev = TS(j2);
                        vprev = vj;
                        ++m;
                    }
                    if (!is_long) {
                        double vh = lin_value_at(hi, j2, ts0, tsl, w0, wl, TS, W);
                        tot = __dadd_rn(tot, lin_piece(vprev, vh, hi - prev));
                    }
                }
                if (is_long) push_long(p, j, k);
                else p.out[j][oidx] = __ddiv_rn(tot, US_PER_S);
            }
        }
        __syncthreads();  // stage buffers free for the next TMA
    }
}

// ------------------------------------------------------------ K3 tile scan
constexpr int SCAN_THREADS = 1024;
__global__ void __launch_bounds__(SCAN_THREADS) tile_scan_kernel(AttrParams p) {
    __shared__ unsigned long long s[SCAN_THREADS][2];
    const int tid = threadIdx.x;
    const int64_t n = p.ntiles;
    const int64_t per = ceil_div(n, SCAN_THREADS);
    const int64_t b0 = min(n, tid * per), b1 = min(n, b0 + per);
    i128 local = 0;
    for (int64_t b = b0; b < b1; ++b) local += join(p.tile_fx[2 * b], p.tile_fx[2 * b + 1]);
    I128Parts lp = split(local);
    s[tid][0] = lp.lo;
    s[tid][1] = lp.hi;
    __syncthreads();
    // Hillis-Steele inclusive scan over per-thread sums
    for (int off = 1; off < SCAN_THREADS; off <<= 1) {
        i128 v = join(s[tid][0], s[tid][1]);
        i128 add = tid >= off ? join(s[tid - off][0], s[tid - off][1]) : (i128)0;
        __syncthreads();
        I128Parts q = split(v + add);
        s[tid][0] = q.lo;
        s[tid][1] = q.hi;
        __syncthreads();
    }
    i128 run = tid ? join(s[tid - 1][0], s[tid - 1][1]) : (i128)0;
    for (int64_t b = b0; b < b1; ++b) {
        I128Parts q = split(run);
        p.prefix[2 * b] = q.lo;
        p.prefix[2 * b + 1] = q.hi;
        run += join(p.tile_fx[2 * b], p.tile_fx[2 * b + 1]);
    }
    if (tid == SCAN_THREADS - 1) {
        I128Parts q = split(join(s[tid][0], s[tid][1]));
        p.prefix[2 * n] = q.lo;
        p.prefix[2 * n + 1] = q.hi;
    }
}

// ------------------------------------------------------ K4 long intervals
template <int KIND>
__device__ __forceinline__ double term_global(const AttrParams &p, int64_t i) {
    auto TS = [&](int64_t g) -> int64_t { return g < p.S ? __ldg(p.ts + g) : p.span_hi; };
    auto W = [&](int64_t g) -> double { return __ldg(p.w + g); };
    if (KIND == DW_SIGNAL_STEP) return __dmul_rn(W(i), (double)(TS(i + 1) - TS(i)));
    double va = lin_sample_value(i, p.S, TS, W);
    double vb = lin_sample_value(i + 1, p.S, TS, W);
    return lin_piece(va, vb, TS(i + 1) - TS(i));
}

// exact sum of terms [j0, j1] (inclusive), whole warp participates
template <int KIND>
__device__ i128 range_sum(const AttrParams &p, int64_t j0, int64_t j1) {
    const int lane = threadIdx.x & 31;
    if (j1 < j0) return 0;
    auto span_sum = [&](int64_t a, int64_t b) -> i128 {
        i128 acc = 0;
        for (int64_t i = a + lane; i <= b; i += 32) acc += q_term(term_global<KIND>(p, i));
        return warp_sum_i128(acc);
    };
    const int64_t ta = j0 / TILE, tb = j1 / TILE;
    if (ta == tb) return span_sum(j0, j1);
    i128 s = span_sum(j0, (ta + 1) * TILE - 1) + span_sum(tb * TILE, j1);
    s += join(p.prefix[2 * tb], p.prefix[2 * tb + 1]) -
         join(p.prefix[2 * (ta + 1)], p.prefix[2 * (ta + 1) + 1]);
    return s;
}

__device__ __forceinline__ int64_t lower_bound_g(const int64_t *a, int64_t n, int64_t key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = lo + ((hi - lo) >> 1);
        if (__ldg(a + mid) < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ int64_t upper_bound_g(const int64_t *a, int64_t n, int64_t key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = lo + ((hi - lo) >> 1);
        if (__ldg(a + mid) <= key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

template <int KIND>
__global__ void __launch_bounds__(256) long_intervals_kernel(AttrParams p) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
    const int64_t count = (int64_t)p.st->long_count;
    const int64_t S = p.S;
    auto TS = [&](int64_t g) -> int64_t { return g < S ? __ldg(p.ts + g) : p.span_hi; };
    auto W = [&](int64_t g) -> double { return __ldg(p.w + g); };
    for (int64_t e = warp; e < count; e += nwarps) {
        unsigned long long ent = p.long_list[e];
        int j = (int)(ent >> 56);
        int64_t k = (int64_t)(ent & ((1ULL << 56) - 1));
        int64_t lo = __ldg(p.start[j] + k), hi = __ldg(p.end[j] + k);
        i128 acc;
        if (KIND == DW_SIGNAL_STEP) {
            int64_t a = upper_bound_g(p.ts, S, lo) - 1;
            int64_t b = lower_bound_g(p.ts, S, hi) - 1;
            acc = range_sum<KIND>(p, a + 1, b - 1);
            if (lane == 0) {
                acc += q_term(__dmul_rn(W(a), (double)(TS(a + 1) - lo)));
                acc += q_term(__dmul_rn(W(b), (double)(min(TS(b + 1), hi) - TS(b))));
            }
        } else {
            int64_t first = upper_bound_g(p.ts, S, lo);
            int64_t last = lower_bound_g(p.ts, S, hi);
            acc = range_sum<KIND>(p, first, last - 2);
            if (lane == 0) {
                int64_t lbj = (first > 0 && TS(first - 1) == lo) ? first - 1 : first;
                double vlo = lin_value_at(lo, lbj, TS(0), TS(S - 1), W(0), W(S - 1), TS, W);
                double vf = lin_sample_value(first, S, TS, W);
                acc += q_term(lin_piece(vlo, vf, TS(first) - lo));
                double vl = lin_sample_value(last - 1, S, TS, W);
                double vh = lin_value_at(hi, last, TS(0), TS(S - 1), W(0), W(S - 1), TS, W);
                acc += q_term(lin_piece(vl, vh, hi - TS(last - 1)));
            }
        }
        if (lane == 0) {
            int64_t oidx = p.perm[j] ? __ldg(p.perm[j] + k) : k;
            p.out[j][oidx] = term_fx_to_joules(acc);
        }
    }
}

// ------------------------------------------------------- K5 sums / finalize
constexpr int SUM_THREADS = 512;
// Exact fixed-point sum (2^-64 J) with the last-block-done pattern.
__global__ void __launch_bounds__(SUM_THREADS) fx_sum_kernel(const double *x, int64_t n,
                                                             unsigned long long *partials,
                                                             unsigned int *done, double *out) {
    __shared__ unsigned long long red[SUM_THREADS / 32][2];
    __shared__ bool last;
    i128 acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)SUM_THREADS + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * SUM_THREADS)
        acc += fx_from_double(__ldg(x + i), FX_JOULE_BITS);
    acc = warp_sum_i128(acc);
    if ((threadIdx.x & 31) == 0) {
        I128Parts pp = split(acc);
        red[threadIdx.x >> 5][0] = pp.lo;
        red[threadIdx.x >> 5][1] = pp.hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        i128 s = 0;
        for (int k = 0; k < SUM_THREADS / 32; ++k) s += join(red[k][0], red[k][1]);
        I128Parts pp = split(s);
        partials[2 * blockIdx.x] = pp.lo;
        partials[2 * blockIdx.x + 1] = pp.hi;
        __threadfence();
        unsigned int ticket = atomicAdd(done, 1u);
        last = ticket == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        i128 s = 0;
        for (unsigned b = 0; b < gridDim.x; ++b)
            s += join(((volatile unsigned long long *)partials)[2 * b],
                      ((volatile unsigned long long *)partials)[2 * b + 1]);
        *out = fx_to_double(s, FX_JOULE_BITS);
        *done = 0;  // reusable
    }
}

// total over the whole span + idle (energy.py:318-324)
template <int KIND>
__global__ void ledger_finalize_kernel(AttrParams p, const double *op_total) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int64_t S = p.S;
    const int64_t nterms = KIND == DW_SIGNAL_STEP ? S : (S > 1 ? S - 1 : 1);
    double total;
    if (nterms <= DIRECT) {
        // reference-literal sequential sum over the span
        auto TS = [&](int64_t g) -> int64_t { return g < S ? p.ts[g] : p.span_hi; };
        auto W = [&](int64_t g) -> double { return p.w[g]; };
        double t = 0.0;
        if (KIND == DW_SIGNAL_STEP) {
            for (int64_t i = 0; i < S; ++i) t = __dadd_rn(t, __dmul_rn(W(i), (double)(TS(i + 1) - TS(i))));
        } else if (S == 1) {
            t = 0.0;
        } else {
            for (int64_t i = 0; i + 1 < S; ++i)
                t = __dadd_rn(t, lin_piece(lin_sample_value(i, S, TS, W),
                                           lin_sample_value(i + 1, S, TS, W), TS(i + 1) - TS(i)));
        }
        total = __ddiv_rn(t, US_PER_S);
    } else {
        total = term_fx_to_joules(join(p.prefix[2 * p.ntiles], p.prefix[2 * p.ntiles + 1]));
    }
    double opt = op_total ? *op_total : 0.0;
    p.st->totals[0] = total;
    p.st->totals[1] = opt;
    double idle = total - opt;
    p.st->totals[2] = idle > 0.0 ? idle : 0.0;
}

// unsorted sets: gather (start, end) into sorted order
__global__ void gather_sorted_kernel(const int64_t *perm, const int64_t *end, int64_t n,
                                     int64_t *end_sorted) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) end_sorted[i] = __ldg(end + __ldg(perm + i));
}
__global__ void iota_kernel(int64_t *a, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] = i;
}

// --------------------------------------------------------- sampler read
__global__ void step_value_at_kernel(const int64_t *ts, const double *w, int64_t S,
                                     int64_t span_hi, const double *t, int64_t m, double *out) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m) return;
    // PowerSignal.value_at (energy.py:57-66): clamp to the span, then the
    // segment with s <= t < e; t == end falls through to the last watts.
    double lo = (double)__ldg(ts), hi = (double)span_hi;
    double x = __ldg(t + k);
    x = fmin(fmax(x, lo), hi);
    int64_t l = 0, h = S;  // last i with ts[i] <= x
    while (l < h) {
        int64_t mid = (l + h) >> 1;
        if ((double)__ldg(ts + mid) <= x) l = mid + 1; else h = mid;
    }
    int64_t i = l - 1;
    if (i < 0) i = 0;
    out[k] = __ldg(w + i);
}

// ================================================================ host side
static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct AttrLayout {
    size_t status, first, tile_fx, prefix, long_list, sum_partials, sum_done, sum_out;
    size_t sort_keys[DW_MAX_SETS], sort_perm[DW_MAX_SETS], sort_end[DW_MAX_SETS],
        sort_iota[DW_MAX_SETS];
    size_t cub_tmp, cub_bytes, total;
};

constexpr int SUM_BLOCKS = 1024;

static size_t cub_sort_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int64_t *)nullptr, (int64_t *)nullptr,
                                    (const int64_t *)nullptr, (int64_t *)nullptr, (int)n);
    return bytes;
}

static AttrLayout attr_layout(int64_t S, const int64_t *sizes, const int32_t *sorted, int nsets) {
    AttrLayout L{};
    int64_t ntiles = S > 0 ? ceil_div(S, TILE) : 0;
    int64_t nint = 0;
    for (int j = 0; j < nsets; ++j) nint += sizes[j];
    size_t off = 0;
    L.status = off; off += align_up(STATUS_BYTES);
    L.first = off; off += align_up(sizeof(int64_t) * (size_t)(ntiles + 1) * DW_MAX_SETS);
    L.tile_fx = off; off += align_up(16 * (size_t)(ntiles + 1));
    L.prefix = off; off += align_up(16 * (size_t)(ntiles + 2));
    L.long_list = off; off += align_up(8 * (size_t)(nint + 1));
    L.sum_partials = off; off += align_up(16 * (size_t)SUM_BLOCKS);
    L.sum_done = off; off += align_up(16);
    L.sum_out = off; off += align_up(16);
    size_t cub = 0;
    for (int j = 0; j < nsets; ++j) {
        if (sorted && sorted[j]) continue;
        size_t n = (size_t)sizes[j];
        L.sort_keys[j] = off; off += align_up(8 * n);
        L.sort_perm[j] = off; off += align_up(8 * n);
        L.sort_end[j] = off; off += align_up(8 * n);
        L.sort_iota[j] = off; off += align_up(8 * n);
        size_t c = cub_sort_bytes(sizes[j]);
        if (c > cub) cub = c;
    }
    L.cub_tmp = off;
    L.cub_bytes = cub;
    off += align_up(cub);
    L.total = off;
    return L;
}

static bool aligned16(const void *p) { return ((uintptr_t)p & 15) == 0; }

static int attribute_impl(const dw_signal_t *sig, dw_interval_set_t *sets, int nsets,
                          void *ws, size_t ws_bytes, cudaStream_t stream, bool ledger,
                          dw_interval_set_t *ops_for_total) {
    if (!sig || nsets < 0 || nsets > DW_MAX_SETS || (nsets && !sets) || !ws) return DW_E_ARG;
    if (sig->kind != DW_SIGNAL_STEP && sig->kind != DW_SIGNAL_LINEAR) return DW_E_ARG;
    if (!aligned16(ws)) return DW_E_ARG;
    int64_t sizes[DW_MAX_SETS] = {0};
    int32_t sorted[DW_MAX_SETS] = {0};
    for (int j = 0; j < nsets; ++j) {
        if (sets[j].n < 0) return DW_E_ARG;
        if (sets[j].n && (!sets[j].d_start || !sets[j].d_end || !sets[j].d_joules)) return DW_E_ARG;
        sizes[j] = sets[j].n;
        sorted[j] = sets[j].sorted;
    }
    const int64_t S = sig->n;
    AttrLayout L = attr_layout(S, sizes, sorted, nsets);
    if (ws_bytes < L.total) return DW_E_WORKSPACE;
    char *base = (char *)ws;
    DevStatus *st = (DevStatus *)(base + L.status);
    status_init_kernel<<<1, 32, 0, stream>>>(st);
    count_launch();
    if (S <= 0 || !sig->d_ts || !sig->d_watts) {
        // SignalError("empty power signal"): flag through the order slot
        DW_CHECK_LAUNCH();
        return DW_E_EMPTY;
    }
    if (!aligned16(sig->d_ts) || !aligned16(sig->d_watts)) return DW_E_ARG;

    AttrParams p{};
    p.ts = sig->d_ts;
    p.w = sig->d_watts;
    p.S = S;
    p.span_hi = sig->kind == DW_SIGNAL_STEP ? sig->span_hi : 0;
    p.ntiles = ceil_div(S, TILE);
    p.kind = sig->kind;
    p.nsets = nsets;
    p.validate_order = sig->validate_order;
    p.first = (const int64_t *)(base + L.first);
    p.tile_fx = (unsigned long long *)(base + L.tile_fx);
    p.prefix = (unsigned long long *)(base + L.prefix);
    p.long_list = (unsigned long long *)(base + L.long_list);
    p.st = st;
    for (int j = 0; j < nsets; ++j) {
        p.n[j] = sets[j].n;
        p.out[j] = sets[j].d_joules;
        if (sets[j].sorted || sets[j].n == 0) {
            p.start[j] = sets[j].d_start;
            p.end[j] = sets[j].d_end;
            p.perm[j] = nullptr;
            p.check_sorted[j] = sets[j].n > 1;
        } else {
            int64_t n = sets[j].n;
            int64_t *keys = (int64_t *)(base + L.sort_keys[j]);
            int64_t *perm = (int64_t *)(base + L.sort_perm[j]);
            int64_t *endv = (int64_t *)(base + L.sort_end[j]);
            int64_t *iota = (int64_t *)(base + L.sort_iota[j]);
            iota_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, stream>>>(iota, n);
            count_launch();
            size_t cub_bytes = L.cub_bytes;
            cub::DeviceRadixSort::SortPairs(base + L.cub_tmp, cub_bytes, sets[j].d_start, keys,
                                            iota, perm, (int)n, 0, 64, stream);
            count_launch(4);
            gather_sorted_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, stream>>>(perm, sets[j].d_end,
                                                                                 n, endv);
            count_launch();
            p.start[j] = keys;
            p.end[j] = endv;
            p.perm[j] = perm;
            p.check_sorted[j] = 0;
        }
    }

    const int64_t nb = (p.ntiles + 1) * (int64_t)nsets;
    if (nb > 0) {
        partition_kernel<<<(unsigned)ceil_div(nb, 256), 256, 0, stream>>>(p);
        count_launch();
    }
    const size_t smem = sizeof(TileSmem);
    int grid = (int)std::min<int64_t>(p.ntiles, (int64_t)num_sms() * 3);
    if (sig->kind == DW_SIGNAL_STEP) {
        cudaFuncSetAttribute(attribute_tiles_kernel<DW_SIGNAL_STEP>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attribute_tiles_kernel<DW_SIGNAL_STEP><<<grid, ATTR_THREADS, smem, stream>>>(p);
    } else {
        cudaFuncSetAttribute(attribute_tiles_kernel<DW_SIGNAL_LINEAR>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attribute_tiles_kernel<DW_SIGNAL_LINEAR><<<grid, ATTR_THREADS, smem, stream>>>(p);
    }
    count_launch();
    tile_scan_kernel<<<1, SCAN_THREADS, 0, stream>>>(p);
    count_launch();
    const int long_grid = num_sms() * 4;
    if (sig->kind == DW_SIGNAL_STEP)
        long_intervals_kernel<DW_SIGNAL_STEP><<<long_grid, 256, 0, stream>>>(p);
    else
        long_intervals_kernel<DW_SIGNAL_LINEAR><<<long_grid, 256, 0, stream>>>(p);
    count_launch();

    if (ledger) {
        double *op_total = nullptr;
        if (ops_for_total && ops_for_total->n > 0) {
            op_total = (double *)(base + L.sum_out);
            unsigned blocks = (unsigned)std::min<int64_t>(SUM_BLOCKS, ceil_div(ops_for_total->n, SUM_THREADS));
            cudaMemsetAsync(base + L.sum_done, 0, 16, stream);
            fx_sum_kernel<<<blocks, SUM_THREADS, 0, stream>>>(
                ops_for_total->d_joules, ops_for_total->n, (unsigned long long *)(base + L.sum_partials),
                (unsigned int *)(base + L.sum_done), op_total);
            count_launch();
        }
        if (sig->kind == DW_SIGNAL_STEP)
            ledger_finalize_kernel<DW_SIGNAL_STEP><<<1, 32, 0, stream>>>(p, op_total);
        else
            ledger_finalize_kernel<DW_SIGNAL_LINEAR><<<1, 32, 0, stream>>>(p, op_total);
        count_launch();
    }
    DW_CHECK_LAUNCH();
    return DW_OK;
}

}  // namespace dw

using namespace dw;

extern "C" {

size_t dw_attribute_workspace_size(int64_t n_samples, const int64_t *set_sizes, int32_t nsets) {
    if (nsets < 0 || nsets > DW_MAX_SETS) return 0;
    int64_t sizes[DW_MAX_SETS] = {0};
    int32_t sorted[DW_MAX_SETS] = {0};  // worst case: every set needs sorting
    for (int j = 0; j < nsets; ++j) sizes[j] = set_sizes ? set_sizes[j] : 0;
    return attr_layout(n_samples, sizes, sorted, nsets).total;
}

int dw_attribute(const dw_signal_t *sig, dw_interval_set_t *sets, int32_t nsets, void *d_workspace,
                 size_t workspace_bytes, dw_stream_t stream) {
    return attribute_impl(sig, sets, nsets, d_workspace, workspace_bytes, (cudaStream_t)stream,
                          false, nullptr);
}

int dw_ledger(const dw_signal_t *sig, dw_interval_set_t *ops, dw_interval_set_t *kernels,
              void *d_workspace, size_t workspace_bytes, dw_stream_t stream) {
    if (!ops || !kernels) return DW_E_ARG;
    dw_interval_set_t sets[2] = {*ops, *kernels};
    return attribute_impl(sig, sets, 2, d_workspace, workspace_bytes, (cudaStream_t)stream, true,
                          &sets[0]);
}

int dw_status(const void *d_workspace, dw_stream_t stream, dw_status_t *out) {
    if (!d_workspace || !out) return DW_E_ARG;
    DevStatus st;
    if (cudaMemcpyAsync(&st, d_workspace, sizeof(st), cudaMemcpyDeviceToHost,
                        (cudaStream_t)stream) != cudaSuccess)
        return DW_E_CUDA;
    if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return DW_E_CUDA;
    auto idx = [](unsigned long long v) -> int64_t {
        return v == (unsigned long long)NONE ? -1 : (int64_t)v;
    };
    out->code = DW_OK;
    out->bad_set = -1;
    for (int j = 0; j < DW_MAX_SETS; ++j) {
        out->bad_index[j] = idx(st.bad_index[j]);
        out->unsorted_index[j] = idx(st.unsorted_index[j]);
    }
    out->order_index = idx(st.order_index);
    out->long_intervals = (int64_t)st.long_count;
    for (int k = 0; k < 4; ++k) out->totals[k] = st.totals[k];
    if (out->order_index >= 0) {
        out->code = DW_E_ORDER;
    } else {
        for (int j = 0; j < DW_MAX_SETS; ++j)
            if (out->unsorted_index[j] >= 0) { out->code = DW_E_UNSORTED; out->bad_set = j; break; }
        if (out->code == DW_OK)
            for (int j = 0; j < DW_MAX_SETS; ++j)
                if (out->bad_index[j] >= 0) { out->code = DW_E_SPAN; out->bad_set = j; break; }
    }
    return out->code;
}

size_t dw_fx_sum_workspace_size(int64_t n) {
    (void)n;
    return 16 * (size_t)SUM_BLOCKS + 256;
}

int dw_fx_sum(const double *d_x, int64_t n, double *d_out, void *d_workspace, size_t ws_bytes,
              dw_stream_t stream) {
    if (n < 0 || !d_out || !d_workspace || ws_bytes < dw_fx_sum_workspace_size(n)) return DW_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    char *base = (char *)d_workspace;
    if (n == 0) {
        cudaMemsetAsync(d_out, 0, sizeof(double), s);
        DW_CHECK_LAUNCH();
        return DW_OK;
    }
    unsigned blocks = (unsigned)std::min<int64_t>(SUM_BLOCKS, ceil_div(n, SUM_THREADS));
    unsigned int *done = (unsigned int *)(base + 16 * (size_t)SUM_BLOCKS);
    cudaMemsetAsync(done, 0, 16, s);
    fx_sum_kernel<<<blocks, SUM_THREADS, 0, s>>>(d_x, n, (unsigned long long *)base, done, d_out);
    count_launch();
    DW_CHECK_LAUNCH();
    return DW_OK;
}

int dw_step_value_at(const dw_signal_t *sig, const double *d_t, int64_t m, double *d_out,
                     dw_stream_t stream) {
    if (!sig || sig->n <= 0 || m < 0 || (m && (!d_t || !d_out))) return DW_E_ARG;
    if (m == 0) return DW_OK;
    step_value_at_kernel<<<(unsigned)ceil_div(m, 256), 256, 0, (cudaStream_t)stream>>>(
        sig->d_ts, sig->d_watts, sig->n, sig->span_hi, d_t, m, d_out);
    count_launch();
    DW_CHECK_LAUNCH();
    return DW_OK;
}

}  // extern "C"
