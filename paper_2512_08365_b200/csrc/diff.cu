// diff.cu -- cross-system differential diff and ranking on B200 (sm_100a).
//
//   K4 detect_pairs   detect_waste's per-pair rule over CSR segment pairs
//                     (detect.py:72-130): CPython-3.12 sum() of member joules,
//                     latency = max end - min start, ratio / side / verdict /
//                     informational / wasted, plus the report ranking key.
//   K5 join           signature hash-join: shared
//                     open-addressing table sig -> dense id, stable radix sort of
//                     each side by id (time order kept), k-th occurrence pairing,
//                     fused deltas + verdict + key + key histogram.
//   K6 rank           report order (detect.py:263-266): top-k by the 128-bit key
//                     (waste flag | wasted bits, ~tie) -- radix-select on the key
//                     histogram, compaction of the candidates, CUB sort of the
//                     (few) candidates.  Also the exact wasted-joules sum.
#include <algorithm>

#include <cub/cub.cuh>

#include "dw_common.cuh"

namespace dw {

constexpr int8_t V_BELOW = 0, V_TRADEOFF = 1, V_WASTE = 2;
constexpr int8_t SIDE_NONE = 0, SIDE_A = 1, SIDE_B = 2;
constexpr double LATENCY_SLACK = 1.01;      // detect.py:24
constexpr double OUTPUT_DIFF_LIMIT = 0.01;  // detect.py:25
constexpr double THRESHOLD_FLOOR = 0.05;    // detect.py:23

constexpr int HIST_BITS = 8;
constexpr int HIST_BINS = 1 << HIST_BITS;

// ranking key: descending (hi, lo) == report order.  hi = waste flag | bits of
// wasted_joules (>= 0, so the bit pattern is monotone; -0.0 folds onto +0.0);
// lo = ~((tie + 1) << 32 | finding index): ascending nodes_a, then input order
// (Python's sort is stable).
__device__ __forceinline__ uint64_t key_hi(int8_t verdict, double wasted) {
    uint64_t b = (uint64_t)__double_as_longlong(wasted) & 0x7FFFFFFFFFFFFFFFULL;
    return (verdict == V_WASTE ? 0x8000000000000000ULL : 0ULL) | b;
}
__device__ __forceinline__ uint64_t key_lo(int64_t tie, int64_t idx) {
    return ~((((uint64_t)(tie + 1)) << 32) | ((uint64_t)idx & 0xFFFFFFFFULL));
}

struct Verdict {
    double ratio, wasted;
    int8_t verdict, side, info;
};

// detect.py:93-126 for one pair
__device__ __forceinline__ Verdict judge(double ea, double eb, int64_t la, int64_t lb,
                                        double out_diff, double threshold) {
    Verdict v;
    const double high = ea >= eb ? ea : eb, low = ea >= eb ? eb : ea;
    if (high == low) {
        v.ratio = 1.0;
        v.side = SIDE_NONE;
    } else {
        v.ratio = low > 0 ? __ddiv_rn(high, low) : __longlong_as_double(0x7FF0000000000000LL);
        v.side = ea > eb ? SIDE_A : SIDE_B;
    }
    if (v.ratio >= __dadd_rn(1.0, threshold)) {
        const int64_t eff = v.side == SIDE_A ? lb : la, ineff = v.side == SIDE_A ? la : lb;
        v.verdict = ((double)eff <= __dmul_rn(LATENCY_SLACK, (double)ineff) && out_diff <= OUTPUT_DIFF_LIMIT)
                        ? V_WASTE
                        : V_TRADEOFF;
    } else {
        v.verdict = V_BELOW;
    }
    v.info = v.verdict == V_BELOW && v.ratio >= __dadd_rn(1.0, THRESHOLD_FLOOR);
    v.wasted = __dsub_rn(high, low);
    return v;
}

struct FindCols {
    double *ea, *eb, *ratio, *wasted;
    int64_t *la, *lb;
    int8_t *verdict, *side, *info;
    uint64_t *khi, *klo;
};

__device__ __forceinline__ void store_finding(const FindCols &o, int64_t f, double ea, double eb,
                                              int64_t la, int64_t lb, const Verdict &v,
                                              int64_t tie) {
    if (o.ea) o.ea[f] = ea;
    if (o.eb) o.eb[f] = eb;
    if (o.ratio) o.ratio[f] = v.ratio;
    if (o.la) o.la[f] = la;
    if (o.lb) o.lb[f] = lb;
    if (o.verdict) o.verdict[f] = v.verdict;
    if (o.side) o.side[f] = v.side;
    if (o.info) o.info[f] = v.info;
    if (o.wasted) o.wasted[f] = v.wasted;
    o.khi[f] = key_hi(v.verdict, v.wasted);
    o.klo[f] = key_lo(tie, f);
}

static FindCols cols_of(const dw_findings_t *f) {
    FindCols c;
    c.ea = f->d_energy_a;
    c.eb = f->d_energy_b;
    c.ratio = f->d_ratio;
    c.wasted = f->d_wasted;
    c.la = f->d_latency_a;
    c.lb = f->d_latency_b;
    c.verdict = f->d_verdict;
    c.side = f->d_side;
    c.info = f->d_informational;
    c.khi = f->d_key_hi;
    c.klo = f->d_key_lo;
    return c;
}

// ------------------------------------------------------------- K4 CSR pairs
__global__ void detect_pairs_kernel(int64_t P, const int64_t *off_a, const int32_t *mem_a,
                                    const int64_t *off_b, const int32_t *mem_b,
                                    const double *ja, const double *jb, const int64_t *sa,
                                    const int64_t *ea_, const int64_t *sb, const int64_t *eb_,
                                    const double *out_diff, const int64_t *tie, double threshold,
                                    FindCols o) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= P) return;
    PySum su_a, su_b;
    int64_t smin = 0, emax = 0;
    const int64_t a0 = off_a[p], a1 = off_a[p + 1];
    for (int64_t k = a0; k < a1; ++k) {
        const int32_t m = mem_a[k];
        su_a.add(ja[m]);
        const int64_t s = sa[m], e = ea_[m];
        if (k == a0 || s < smin) smin = s;
        if (k == a0 || e > emax) emax = e;
    }
    const int64_t la = a1 > a0 ? emax - smin : 0;
    const int64_t b0 = off_b[p], b1 = off_b[p + 1];
    for (int64_t k = b0; k < b1; ++k) {
        const int32_t m = mem_b[k];
        su_b.add(jb[m]);
        const int64_t s = sb[m], e = eb_[m];
        if (k == b0 || s < smin) smin = s;
        if (k == b0 || e > emax) emax = e;
    }
    const int64_t lb = b1 > b0 ? emax - smin : 0;
    const double e_a = su_a.result(), e_b = su_b.result();
    const Verdict v = judge(e_a, e_b, la, lb, out_diff ? out_diff[p] : 0.0, threshold);
    store_finding(o, p, e_a, e_b, la, lb, v, tie ? tie[p] : 0);
}

// ------------------------------------------------------------------ K6 rank
struct RankParams {
    const uint64_t *khi, *klo;
    int64_t P, k;
    unsigned int *hist;        // [HIST_BINS]
    unsigned long long *sel;   // [2]: bin, count strictly above the bin
    unsigned long long *cand_n;
    uint64_t *cand_hi, *cand_lo;
    int64_t *cand_idx;
    int64_t cand_cap;
    int pos;                   // bit position of the current digit in the 128-bit key
    uint64_t phi, plo, mhi, mlo;  // prefix fixed so far and its mask
};

__device__ __forceinline__ unsigned digit128(uint64_t hi, uint64_t lo, int pos) {
    return pos >= 64 ? (unsigned)((hi >> (pos - 64)) & (HIST_BINS - 1))
                     : (unsigned)((lo >> pos) & (HIST_BINS - 1));
}

__global__ void rank_hist_kernel(RankParams r) {
    __shared__ unsigned int h[HIST_BINS];
    for (int b = threadIdx.x; b < HIST_BINS; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const bool need_lo = r.pos < 64 || r.mlo;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r.P;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t hi = r.khi[i];
        if ((hi & r.mhi) != r.phi) continue;
        const uint64_t lo = need_lo ? r.klo[i] : 0;
        if ((lo & r.mlo) != r.plo) continue;
        atomicAdd(&h[digit128(hi, lo, r.pos)], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < HIST_BINS; b += blockDim.x)
        if (h[b]) atomicAdd(&r.hist[b], h[b]);
}

// Walk the histogram from the top bin down to the bin holding the need-th
// largest key of the current prefix.  sel = {bin, keys strictly above it}.
__global__ void rank_select_kernel(RankParams r, int64_t need) {
    if (threadIdx.x != 0) return;
    int64_t above = 0;
    int b = HIST_BINS - 1;
    for (; b > 0; --b) {
        if (above + (int64_t)r.hist[b] >= need) break;
        above += r.hist[b];
    }
    r.sel[0] = (unsigned long long)b;
    r.sel[1] = (unsigned long long)above;
}

// copy every key >= (thr_hi, thr_lo) into the candidate buffer
__global__ void rank_compact_kernel(RankParams r, uint64_t thr_hi, uint64_t thr_lo) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r.P;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t hi = r.khi[i];
        if (hi < thr_hi) continue;
        const uint64_t lo = r.klo[i];
        if (hi == thr_hi && lo < thr_lo) continue;
        unsigned long long slot = atomicAdd(r.cand_n, 1ULL);
        if ((int64_t)slot < r.cand_cap) {
            r.cand_hi[slot] = hi;
            r.cand_lo[slot] = lo;
            r.cand_idx[slot] = i;
        }
    }
}

__global__ void gather_u64_kernel(const uint64_t *src, const int64_t *idx, int64_t n, uint64_t *dst) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[idx[i]];
}
__global__ void gather_i64_kernel(const int64_t *src, const int64_t *idx, int64_t n, int64_t *dst) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[idx[i]];
}
__global__ void iota64_kernel(int64_t *a, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] = i;
}

// n_waste, exact wasted sum over waste findings, n
__global__ void waste_sum_kernel(const uint64_t *khi, int64_t P, unsigned long long *partials,
                                 unsigned int *done, double *summary) {
    __shared__ unsigned long long red[8][3];
    __shared__ bool last;
    i128 acc = 0;
    unsigned long long cnt = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = khi[i];
        if (k >> 63) {
            acc += fx_from_double(__longlong_as_double((long long)(k & 0x7FFFFFFFFFFFFFFFULL)),
                                  FX_JOULE_BITS);
            ++cnt;
        }
    }
    acc = warp_sum_i128(acc);
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0) {
        I128Parts q = split(acc);
        red[threadIdx.x >> 5][0] = q.lo;
        red[threadIdx.x >> 5][1] = q.hi;
        red[threadIdx.x >> 5][2] = cnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        i128 s = 0;
        unsigned long long c = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            s += join(red[w][0], red[w][1]);
            c += red[w][2];
        }
        I128Parts q = split(s);
        partials[3 * blockIdx.x] = q.lo;
        partials[3 * blockIdx.x + 1] = q.hi;
        partials[3 * blockIdx.x + 2] = c;
        __threadfence();
        last = atomicAdd(done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        i128 s = 0;
        unsigned long long c = 0;
        volatile unsigned long long *pp = partials;
        for (unsigned b = 0; b < gridDim.x; ++b) {
            s += join(pp[3 * b], pp[3 * b + 1]);
            c += pp[3 * b + 2];
        }
        summary[0] = (double)c;
        summary[1] = fx_to_double(s, FX_JOULE_BITS);
        summary[2] = (double)P;
        *done = 0;
    }
}

// ------------------------------------------------------------------ K5 join
constexpr uint64_t EMPTY = 0xFFFFFFFFFFFFFFFFULL;

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

struct JoinParams {
    const uint64_t *sig_a, *sig_b;
    int64_t na, nb;
    uint64_t *table;  // [cap] keys
    int32_t *slot_id; // [cap] dense id (1-based; 0 reserved for sig == EMPTY)
    int64_t cap;      // power of two
    int32_t *d_a, *d_b;
    unsigned long long *overflow;
};

__global__ void join_insert_kernel(JoinParams q) {
    const int64_t n = q.na + q.nb;
    const uint64_t mask = (uint64_t)q.cap - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t s = i < q.na ? q.sig_a[i] : q.sig_b[i - q.na];
        if (s == EMPTY) continue;
        uint64_t h = mix64(s) & mask;
        for (int64_t probe = 0;; ++probe) {
            if (probe >= q.cap) {
                atomicAdd(q.overflow, 1ULL);
                break;
            }
            uint64_t k = q.table[h];
            if (k == s) break;
            if (k == EMPTY) {
                uint64_t old = atomicCAS((unsigned long long *)&q.table[h], EMPTY, s);
                if (old == EMPTY || old == s) break;
            }
            h = (h + 1) & mask;
        }
    }
}

__global__ void join_flags_kernel(JoinParams q) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < q.cap;
         i += (int64_t)gridDim.x * blockDim.x)
        q.slot_id[i] = q.table[i] != EMPTY ? 1 : 0;
}

__global__ void join_lookup_kernel(JoinParams q) {
    const int64_t n = q.na + q.nb;
    const uint64_t mask = (uint64_t)q.cap - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t s = i < q.na ? q.sig_a[i] : q.sig_b[i - q.na];
        int32_t id = 0;
        if (s != EMPTY) {
            uint64_t h = mix64(s) & mask;
            while (q.table[h] != s) h = (h + 1) & mask;
            id = q.slot_id[h];  // inclusive scan of occupancy: 1-based
        }
        if (i < q.na) q.d_a[i] = id;
        else q.d_b[i - q.na] = id;
    }
}

// run boundaries of a sorted id column -> first[d], count[d]
__global__ void run_bounds_kernel(const int32_t *dsorted, int64_t n, int64_t *first, int64_t *count) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int32_t d = dsorted[p];
    if (p == 0 || dsorted[p - 1] != d) first[d] = p;
    if (p == n - 1 || dsorted[p + 1] != d) count[d] = p + 1;  // end; turned into a count below
}
__global__ void run_counts_kernel(const int64_t *first, int64_t *count, int64_t D) {
    const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (d >= D) return;
    if (count[d] > 0) count[d] -= first[d];
}

// k-th occurrence pairing over A's sorted order
__global__ void join_pair_kernel(const int32_t *da_sorted, const int64_t *ia_sorted, int64_t na,
                                 const int64_t *first_a, const int64_t *first_b,
                                 const int64_t *count_b, const int64_t *ib_sorted,
                                 int64_t *match_a, int64_t *match_b) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= na) return;
    const int32_t d = da_sorted[p];
    const int64_t t = p - first_a[d];
    const int64_t i = ia_sorted[p];
    int64_t j = -1;
    if (t < count_b[d]) {
        j = ib_sorted[first_b[d] + t];
        match_b[j] = i;
    }
    match_a[i] = j;
}

struct JoinSideDev {
    const int64_t *start, *end, *rank;
    const double *joules, *work;
};

__device__ __forceinline__ double div_or_same(double e, const double *work, int64_t i) {
    return work ? __ddiv_rn(e, work[i]) : e;
}

// findings for A ops (matched or A-only), in A order
__global__ void join_findings_a_kernel(int64_t na, const int64_t *match_a, JoinSideDev A,
                                       JoinSideDev B, double threshold, FindCols o, int64_t *ia,
                                       int64_t *ib, double *epw_a, double *epw_b,
                                       unsigned long long *n_matched) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= na) return;
    const int64_t j = match_a[i];
    const double ea = A.joules[i];
    const int64_t la = A.end[i] - A.start[i];
    double eb = 0.0;
    int64_t lb = 0;
    if (j >= 0) {
        eb = B.joules[j];
        lb = B.end[j] - B.start[j];
    }
    const Verdict v = judge(ea, eb, la, lb, 0.0, threshold);
    store_finding(o, i, ea, eb, la, lb, v, A.rank ? A.rank[i] : i);
    if (ia) ia[i] = i;
    if (ib) ib[i] = j;
    if (epw_a) epw_a[i] = div_or_same(ea, A.work, i);
    if (epw_b) epw_b[i] = j >= 0 ? div_or_same(eb, B.work, j) : 0.0;
    // warp-aggregated matched count
    const unsigned m = __ballot_sync(__activemask(), j >= 0);
    if ((threadIdx.x & 31) == __ffs(__activemask()) - 1) atomicAdd(n_matched, (unsigned long long)__popc(m));
}

__global__ void unmatched_flags_kernel(const int64_t *match_b, int64_t nb, int32_t *flag) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j < nb) flag[j] = match_b[j] < 0 ? 1 : 0;
}

// B-only findings: numbered na + (exclusive rank among unmatched B ops)
__global__ void join_findings_b_kernel(int64_t na, int64_t nb, const int64_t *match_b,
                                       const int32_t *scan_incl, JoinSideDev B, double threshold,
                                       FindCols o, int64_t *ia, int64_t *ib, double *epw_a,
                                       double *epw_b) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= nb || match_b[j] >= 0) return;
    const int64_t f = na + scan_incl[j] - 1;
    const double eb = B.joules[j];
    const int64_t lb = B.end[j] - B.start[j];
    const Verdict v = judge(0.0, eb, 0, lb, 0.0, threshold);
    store_finding(o, f, 0.0, eb, 0, lb, v, -1);  // nodes_a == () sorts first
    if (ia) ia[f] = -1;
    if (ib) ib[f] = j;
    if (epw_a) epw_a[f] = 0.0;
    if (epw_b) epw_b[f] = div_or_same(eb, B.work, j);
}

// ================================================================ host side
static size_t au(size_t x) { return (x + 255) & ~(size_t)255; }

static unsigned blocks_for(int64_t n, int t = 256) {
    int64_t b = (n + t - 1) / t;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)1 << 30));
}

constexpr int64_t CAND_MIN = 1 << 16;

struct RankLayout {
    size_t hist, sel, cand_n, cand_hi, cand_lo, cand_idx, tmp_hi, tmp_lo, tmp_idx, tmp_idx2,
        partials, done, cub, cub_bytes, total;
    int64_t cap;
};

static RankLayout rank_layout(int64_t P, int64_t k) {
    RankLayout L{};
    int64_t cap = std::max<int64_t>(CAND_MIN, 4 * k);
    if (cap > P) cap = P;
    if (cap < 1) cap = 1;
    L.cap = cap;
    size_t off = 0;
    L.hist = off; off += au(4 * HIST_BINS);
    L.sel = off; off += au(64);
    L.cand_n = off; off += au(16);
    L.cand_hi = off; off += au(8 * cap);
    L.cand_lo = off; off += au(8 * cap);
    L.cand_idx = off; off += au(8 * cap);
    L.tmp_hi = off; off += au(8 * cap);
    L.tmp_lo = off; off += au(8 * cap);
    L.tmp_idx = off; off += au(8 * cap);
    L.tmp_idx2 = off; off += au(8 * cap);
    L.partials = off; off += au(24 * 1024);
    L.done = off; off += au(16);
    size_t c1 = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, c1, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                              (const int64_t *)nullptr, (int64_t *)nullptr, (int)cap);
    L.cub = off;
    L.cub_bytes = c1;
    off += au(c1);
    L.total = off;
    return L;
}

// Sort candidates by (hi desc, lo desc), LSD: stable by lo first, then by hi.
static void sort_candidates(char *base, const RankLayout &L, int64_t n, cudaStream_t s) {
    uint64_t *chi = (uint64_t *)(base + L.cand_hi), *clo = (uint64_t *)(base + L.cand_lo);
    int64_t *cidx = (int64_t *)(base + L.cand_idx);
    uint64_t *thi = (uint64_t *)(base + L.tmp_hi), *tlo = (uint64_t *)(base + L.tmp_lo);
    int64_t *tidx = (int64_t *)(base + L.tmp_idx), *tidx2 = (int64_t *)(base + L.tmp_idx2);
    size_t cb = L.cub_bytes;
    // positions 0..n-1 sorted by lo desc
    iota64_kernel<<<blocks_for(n), 256, 0, s>>>(tidx2, n);
    cub::DeviceRadixSort::SortPairsDescending(base + L.cub, cb, clo, tlo, tidx2, tidx, (int)n, 0, 64, s);
    // hi in that order, then stable sort by hi desc carrying positions
    gather_u64_kernel<<<blocks_for(n), 256, 0, s>>>(chi, tidx, n, thi);
    cub::DeviceRadixSort::SortPairsDescending(base + L.cub, cb, thi, chi, tidx, tidx2, (int)n, 0, 64, s);
    // final finding indices
    gather_i64_kernel<<<blocks_for(n), 256, 0, s>>>(cidx, tidx2, n, tidx);
    count_launch(5 + 8);
}

static int rank_impl(int64_t P, const uint64_t *khi, const uint64_t *klo, int64_t k, int64_t *order,
                     double *summary, void *ws, size_t ws_bytes, cudaStream_t s) {
    if (P < 0 || k < 0 || k > P || (P && (!khi || !klo)) || (k && !order) || !ws) return DW_E_ARG;
    RankLayout L = rank_layout(P, k);
    if (ws_bytes < L.total) return DW_E_WORKSPACE;
    char *base = (char *)ws;
    if (summary) {
        cudaMemsetAsync(base + L.done, 0, 16, s);
        if (P > 0) {
            waste_sum_kernel<<<(unsigned)std::min<int64_t>(1024, blocks_for(P)), 256, 0, s>>>(
                khi, P, (unsigned long long *)(base + L.partials), (unsigned int *)(base + L.done),
                summary);
            count_launch();
        } else {
            cudaMemsetAsync(summary, 0, 3 * sizeof(double), s);
        }
    }
    if (k == 0) {
        DW_CHECK_LAUNCH();
        return DW_OK;
    }
    RankParams r{};
    r.khi = khi;
    r.klo = klo;
    r.P = P;
    r.k = k;
    r.hist = (unsigned int *)(base + L.hist);
    r.sel = (unsigned long long *)(base + L.sel);
    r.cand_n = (unsigned long long *)(base + L.cand_n);
    r.cand_hi = (uint64_t *)(base + L.cand_hi);
    r.cand_lo = (uint64_t *)(base + L.cand_lo);
    r.cand_idx = (int64_t *)(base + L.cand_idx);
    r.cand_cap = L.cap;
    // Radix-select the threshold digit by digit (128-bit key, most significant
    // first) until every key >= threshold fits the candidate buffer.
    int64_t need = k;
    uint64_t phi = 0, plo = 0, mhi = 0, mlo = 0;
    uint64_t thr_hi = 0, thr_lo = 0;
    const unsigned grid = (unsigned)std::min<int64_t>(num_sms() * 8, blocks_for(P));
    for (int pos = 128 - HIST_BITS; pos >= 0; pos -= HIST_BITS) {
        r.pos = pos;
        r.phi = phi;
        r.plo = plo;
        r.mhi = mhi;
        r.mlo = mlo;
        cudaMemsetAsync(r.hist, 0, 4 * HIST_BINS, s);
        rank_hist_kernel<<<grid, 512, 0, s>>>(r);
        rank_select_kernel<<<1, 32, 0, s>>>(r, need);
        count_launch(2);
        unsigned long long sel[2];
        cudaMemcpyAsync(sel, r.sel, sizeof(sel), cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) return DW_E_CUDA;
        unsigned int in_bin = 0;
        cudaMemcpy(&in_bin, r.hist + sel[0], 4, cudaMemcpyDeviceToHost);
        const uint64_t dig = sel[0];
        if (pos >= 64) {
            thr_hi = phi | (dig << (pos - 64));
            thr_lo = 0;
        } else {
            thr_hi = phi;
            thr_lo = plo | (dig << pos);
        }
        const int64_t above = (int64_t)sel[1];
        const int64_t candidates = (k - need) + above + (int64_t)in_bin;
        if (candidates <= L.cap || pos == 0) break;
        need -= above;
        phi = thr_hi;
        plo = thr_lo;
        if (pos >= 64) mhi |= ((uint64_t)(HIST_BINS - 1)) << (pos - 64);
        else mlo |= ((uint64_t)(HIST_BINS - 1)) << pos;
    }
    cudaMemsetAsync(r.cand_n, 0, 8, s);
    rank_compact_kernel<<<grid, 256, 0, s>>>(r, thr_hi, thr_lo);
    count_launch();
    unsigned long long nc = 0;
    cudaMemcpyAsync(&nc, r.cand_n, 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if ((int64_t)nc > L.cap) return DW_E_WORKSPACE;  // massive ties at the threshold key
    if ((int64_t)nc < k) return DW_E_ARG;             // cannot happen
    sort_candidates(base, L, (int64_t)nc, s);
    cudaMemcpyAsync(order, base + L.tmp_idx, 8 * k, cudaMemcpyDeviceToDevice, s);
    DW_CHECK_LAUNCH();
    return DW_OK;
}

struct JoinLayout {
    size_t table, slot_id, scan_tmp, scan_bytes, d_a, d_b, ds_a, ds_b, iota_a, iota_b, is_a, is_b,
        first_a, count_a, first_b, count_b, match_a, match_b, flag_b, scan_b, cub, cub_bytes,
        counters, total;
    int64_t cap, D;
};

static int64_t pow2_at_least(int64_t x) {
    int64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

static JoinLayout join_layout(int64_t na, int64_t nb, int64_t max_distinct) {
    JoinLayout L{};
    if (max_distinct <= 0) max_distinct = na + nb;
    L.cap = pow2_at_least(std::max<int64_t>(1024, 2 * std::min<int64_t>(max_distinct, na + nb)));
    L.D = std::min<int64_t>(L.cap, na + nb) + 2;
    size_t off = 0;
    L.table = off; off += au(8 * L.cap);
    L.slot_id = off; off += au(4 * L.cap);
    size_t sb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, sb, (int32_t *)nullptr, (int32_t *)nullptr, (int)L.cap);
    size_t sb2 = 0;
    cub::DeviceScan::InclusiveSum(nullptr, sb2, (int32_t *)nullptr, (int32_t *)nullptr, (int)std::max<int64_t>(nb, 1));
    L.scan_tmp = off;
    L.scan_bytes = std::max(sb, sb2);
    off += au(L.scan_bytes);
    L.d_a = off; off += au(4 * na);
    L.d_b = off; off += au(4 * nb);
    L.ds_a = off; off += au(4 * na);
    L.ds_b = off; off += au(4 * nb);
    L.iota_a = off; off += au(8 * na);
    L.iota_b = off; off += au(8 * nb);
    L.is_a = off; off += au(8 * na);
    L.is_b = off; off += au(8 * nb);
    L.first_a = off; off += au(8 * L.D);
    L.count_a = off; off += au(8 * L.D);
    L.first_b = off; off += au(8 * L.D);
    L.count_b = off; off += au(8 * L.D);
    L.match_a = off; off += au(8 * na);
    L.match_b = off; off += au(8 * nb);
    L.flag_b = off; off += au(4 * nb);
    L.scan_b = off; off += au(4 * nb);
    size_t cs = 0;
    const int64_t nmax = std::max<int64_t>(std::max(na, nb), 1);
    cub::DeviceRadixSort::SortPairs(nullptr, cs, (const int32_t *)nullptr, (int32_t *)nullptr,
                                    (const int64_t *)nullptr, (int64_t *)nullptr, (int)nmax);
    L.cub = off;
    L.cub_bytes = cs;
    off += au(cs);
    L.counters = off; off += au(64);
    L.total = off;
    return L;
}

static int bits_for(int64_t D) {
    int b = 1;
    while (((int64_t)1 << b) <= D) ++b;
    return b;
}

}  // namespace dw

using namespace dw;

extern "C" {

int dw_detect_pairs(int64_t P, const int64_t *d_off_a, const int32_t *d_mem_a, const int64_t *d_off_b,
                    const int32_t *d_mem_b, const double *d_joules_a, const double *d_joules_b,
                    const int64_t *d_start_a, const int64_t *d_end_a, const int64_t *d_start_b,
                    const int64_t *d_end_b, const double *d_out_diff, const int64_t *d_tie,
                    double threshold, dw_findings_t *out, dw_stream_t stream) {
    if (!(threshold > 0.0 && threshold <= 1.0)) return DW_E_ARG;
    if (P < 0 || !out || (P && (!d_off_a || !d_off_b || !out->d_key_hi || !out->d_key_lo)))
        return DW_E_ARG;
    if (P == 0) return DW_OK;
    detect_pairs_kernel<<<blocks_for(P), 256, 0, (cudaStream_t)stream>>>(
        P, d_off_a, d_mem_a, d_off_b, d_mem_b, d_joules_a, d_joules_b, d_start_a, d_end_a,
        d_start_b, d_end_b, d_out_diff, d_tie, threshold, cols_of(out));
    count_launch();
    DW_CHECK_LAUNCH();
    return DW_OK;
}

size_t dw_rank_workspace_size(int64_t P, int64_t k) { return rank_layout(P, k).total; }

int dw_rank(int64_t P, const dw_findings_t *f, int64_t k, int64_t *d_order, double *d_summary,
            void *d_workspace, size_t workspace_bytes, dw_stream_t stream) {
    if (!f) return DW_E_ARG;
    return rank_impl(P, f->d_key_hi, f->d_key_lo, k, d_order, d_summary, d_workspace, workspace_bytes,
                     (cudaStream_t)stream);
}

size_t dw_join_workspace_size(int64_t na, int64_t nb, int64_t max_distinct) {
    return join_layout(na, nb, max_distinct).total;
}

int dw_join_diff(const dw_join_side_t *a, const dw_join_side_t *b, int64_t max_distinct, double threshold,
                 dw_findings_t *out, int64_t *d_ia, int64_t *d_ib, double *d_epw_a, double *d_epw_b,
                 int64_t *d_count, void *d_workspace, size_t workspace_bytes, dw_stream_t stream) {
    if (!(threshold > 0.0 && threshold <= 1.0)) return DW_E_ARG;
    if (!a || !b || !out || !d_count || !d_workspace) return DW_E_ARG;
    const int64_t na = a->n, nb = b->n;
    if (na < 0 || nb < 0 || na + nb >= ((int64_t)1 << 31)) return DW_E_ARG;
    if ((na && (!a->d_sig || !a->d_start || !a->d_end || !a->d_joules)) ||
        (nb && (!b->d_sig || !b->d_start || !b->d_end || !b->d_joules)))
        return DW_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    JoinLayout L = join_layout(na, nb, max_distinct);
    if (workspace_bytes < L.total) return DW_E_WORKSPACE;
    char *base = (char *)d_workspace;
    JoinParams q{};
    q.sig_a = a->d_sig;
    q.sig_b = b->d_sig;
    q.na = na;
    q.nb = nb;
    q.table = (uint64_t *)(base + L.table);
    q.slot_id = (int32_t *)(base + L.slot_id);
    q.cap = L.cap;
    q.d_a = (int32_t *)(base + L.d_a);
    q.d_b = (int32_t *)(base + L.d_b);
    unsigned long long *counters = (unsigned long long *)(base + L.counters);
    q.overflow = counters;
    cudaMemsetAsync(counters, 0, 64, s);
    cudaMemsetAsync(q.table, 0xFF, 8 * L.cap, s);
    const unsigned grid = (unsigned)(num_sms() * 16);
    join_insert_kernel<<<grid, 256, 0, s>>>(q);
    join_flags_kernel<<<grid, 256, 0, s>>>(q);
    size_t sb = L.scan_bytes;
    cub::DeviceScan::InclusiveSum(base + L.scan_tmp, sb, q.slot_id, q.slot_id, (int)L.cap, s);
    join_lookup_kernel<<<grid, 256, 0, s>>>(q);
    count_launch(5);
    const int64_t D = L.D;
    const int nbits = bits_for(D);
    int64_t *first_a = (int64_t *)(base + L.first_a), *count_a = (int64_t *)(base + L.count_a);
    int64_t *first_b = (int64_t *)(base + L.first_b), *count_b = (int64_t *)(base + L.count_b);
    cudaMemsetAsync(count_a, 0, 8 * D, s);
    cudaMemsetAsync(count_b, 0, 8 * D, s);
    int64_t *is_a = (int64_t *)(base + L.is_a), *is_b = (int64_t *)(base + L.is_b);
    int32_t *ds_a = (int32_t *)(base + L.ds_a), *ds_b = (int32_t *)(base + L.ds_b);
    size_t cs = L.cub_bytes;
    if (na) {
        iota64_kernel<<<blocks_for(na), 256, 0, s>>>((int64_t *)(base + L.iota_a), na);
        cub::DeviceRadixSort::SortPairs(base + L.cub, cs, q.d_a, ds_a, (const int64_t *)(base + L.iota_a),
                                        is_a, (int)na, 0, nbits, s);
        run_bounds_kernel<<<blocks_for(na), 256, 0, s>>>(ds_a, na, first_a, count_a);
        count_launch(6);
    }
    if (nb) {
        iota64_kernel<<<blocks_for(nb), 256, 0, s>>>((int64_t *)(base + L.iota_b), nb);
        cub::DeviceRadixSort::SortPairs(base + L.cub, cs, q.d_b, ds_b, (const int64_t *)(base + L.iota_b),
                                        is_b, (int)nb, 0, nbits, s);
        run_bounds_kernel<<<blocks_for(nb), 256, 0, s>>>(ds_b, nb, first_b, count_b);
        count_launch(6);
    }
    run_counts_kernel<<<blocks_for(D), 256, 0, s>>>(first_a, count_a, D);
    run_counts_kernel<<<blocks_for(D), 256, 0, s>>>(first_b, count_b, D);
    int64_t *match_a = (int64_t *)(base + L.match_a), *match_b = (int64_t *)(base + L.match_b);
    cudaMemsetAsync(match_b, 0xFF, 8 * std::max<int64_t>(nb, 1), s);
    if (na)
        join_pair_kernel<<<blocks_for(na), 256, 0, s>>>(ds_a, is_a, na, first_a, first_b, count_b, is_b,
                                                         match_a, match_b);
    count_launch(3);
    JoinSideDev A{a->d_start, a->d_end, a->d_rank, a->d_joules, a->d_work};
    JoinSideDev B{b->d_start, b->d_end, b->d_rank, b->d_joules, b->d_work};
    FindCols o = cols_of(out);
    if (na) {
        join_findings_a_kernel<<<blocks_for(na), 256, 0, s>>>(na, match_a, A, B, threshold, o, d_ia, d_ib,
                                                               d_epw_a, d_epw_b, counters + 1);
        count_launch();
    }
    int32_t *flag_b = (int32_t *)(base + L.flag_b), *scan_b = (int32_t *)(base + L.scan_b);
    if (nb) {
        unmatched_flags_kernel<<<blocks_for(nb), 256, 0, s>>>(match_b, nb, flag_b);
        sb = L.scan_bytes;
        cub::DeviceScan::InclusiveSum(base + L.scan_tmp, sb, flag_b, scan_b, (int)nb, s);
        join_findings_b_kernel<<<blocks_for(nb), 256, 0, s>>>(na, nb, match_b, scan_b, B, threshold, o,
                                                               d_ia, d_ib, d_epw_a, d_epw_b);
        count_launch(4);
    }
    // counts: {P, matched, a_only, b_only} -- assembled on the host side of this call
    unsigned long long host_c[2] = {0, 0};
    int32_t b_only = 0;
    cudaMemcpyAsync(host_c, counters, 16, cudaMemcpyDeviceToHost, s);
    if (nb) cudaMemcpyAsync(&b_only, scan_b + nb - 1, 4, cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return DW_E_CUDA;
    if (host_c[0]) return DW_E_WORKSPACE;  // hash table overflow
    const int64_t matched = (int64_t)host_c[1];
    const int64_t cnt[4] = {na + b_only, matched, na - matched, b_only};
    cudaMemcpyAsync(d_count, cnt, sizeof(cnt), cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    DW_CHECK_LAUNCH();
    return DW_OK;
}

}  // extern "C"
