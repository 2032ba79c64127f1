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
#include <vector>

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
    double *de, *epwr;
    int64_t *dt;
};

// epw_a / epw_b: joules per unit of work of each side (= joules without work)
__device__ __forceinline__ void store_finding(const FindCols &o, int64_t f, double ea, double eb,
                                              int64_t la, int64_t lb, const Verdict &v,
                                              int64_t tie, double epw_a, double epw_b) {
    if (o.de) o.de[f] = __dsub_rn(eb, ea);
    if (o.dt) o.dt[f] = lb - la;
    if (o.epwr) o.epwr[f] = __ddiv_rn(epw_b, epw_a);
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
    if (o.klo) o.klo[f] = key_lo(tie, f);
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
    c.de = f->d_delta_e;
    c.dt = f->d_delta_t;
    c.epwr = f->d_epw_ratio;
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
    store_finding(o, p, e_a, e_b, la, lb, v, tie ? tie[p] : 0, e_a, e_b);
}

// ------------------------------------------------------------------ K6 rank
struct RankParams {
    const uint64_t *khi, *klo;
    const int64_t *tie_rank;   // implicit low keys (klo == NULL): join numbering
    int64_t n_a;
    int64_t P, k;
    unsigned int *hist;        // [HIST_BINS]
    unsigned long long *sel;   // [3]: bin, count strictly above the bin, count in the bin
    unsigned long long *cand_n;
    uint64_t *cand_hi, *cand_lo;
    int64_t *cand_idx;
    int64_t cand_cap;
    int pos;                   // bit position of the current digit in the 128-bit key
    uint64_t phi, plo, mhi, mlo;  // prefix fixed so far and its mask
};

// the low key of finding i: stored, or implied by the join's numbering
// (A findings: tie = rank of the A op; B-only findings: tie = -1)
__device__ __forceinline__ uint64_t lo_of(const RankParams &r, int64_t i) {
    if (r.klo) return r.klo[i];
    const int64_t tie = i < r.n_a ? (r.tie_rank ? r.tie_rank[i] : i) : -1;
    return key_lo(tie, i);
}

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
        const uint64_t lo = need_lo ? lo_of(r, i) : 0;
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
    r.sel[2] = (unsigned long long)r.hist[b];  // keys in the selected bin (one read-back for all three)
}

// copy every key >= (thr_hi, thr_lo) into the candidate buffer
__global__ void rank_compact_kernel(RankParams r, uint64_t thr_hi, uint64_t thr_lo) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r.P;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t hi = r.khi[i];
        if (hi < thr_hi) continue;
        const uint64_t lo = lo_of(r, i);
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

// n_waste, exact wasted sum over waste findings, n; with hist, also the
// rank's first-digit histogram (the top HIST_BITS of key_hi; one read of the
// key column for both)
__global__ void waste_sum_kernel(const uint64_t *khi, int64_t P, unsigned long long *partials,
                                 unsigned int *done, double *summary, unsigned int *hist) {
    __shared__ unsigned long long red[8][3];
    __shared__ unsigned int h[HIST_BINS];
    __shared__ bool last;
    if (hist) {
        for (int b = threadIdx.x; b < HIST_BINS; b += blockDim.x) h[b] = 0;
        __syncthreads();
    }
    i128 acc = 0;
    unsigned long long cnt = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
    // block-uniform trip count: every lane of a warp runs every iteration, so
    // the histogram's warp votes below see full warps
    for (int64_t bb = blockIdx.x * (int64_t)blockDim.x * 4; bb < P; bb += stride) {
        const int64_t b = bb + threadIdx.x;
        uint64_t k[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = b + (int64_t)u * blockDim.x;
            k[u] = i < P ? khi[i] : 0;
        }
        if (hist) {
            // the first digit is the waste flag and the top exponent bits: a
            // warp's keys mostly share one bin, so a warp adds 32 at once
            // instead of 32 same-address shared atomics
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool ok = b + (int64_t)u * blockDim.x < P;
                const unsigned bin = (unsigned)(k[u] >> (64 - HIST_BITS));
                const unsigned b0 = __shfl_sync(0xffffffffu, bin, 0);
                if (__all_sync(0xffffffffu, ok && bin == b0)) {
                    if ((threadIdx.x & 31) == 0) atomicAdd(&h[b0], 32u);
                } else if (ok) {
                    atomicAdd(&h[bin], 1u);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (k[u] >> 63) {
                acc += fx_joules(__longlong_as_double((long long)(k[u] & 0x7FFFFFFFFFFFFFFFULL)));
                ++cnt;
            }
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
    if (hist)
        for (int b = threadIdx.x; b < HIST_BINS; b += blockDim.x)
            if (h[b]) atomicAdd(&hist[b], h[b]);
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
    if (!last) return;
    // the last block sums the partials with all its threads (independent L2 loads)
    __threadfence();
    i128 ps = 0;
    unsigned long long pc = 0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
        ps += join(__ldcg(partials + 3 * b), __ldcg(partials + 3 * b + 1));
        pc += __ldcg(partials + 3 * b + 2);
    }
    ps = warp_sum_i128(ps);
    for (int o = 16; o > 0; o >>= 1) pc += __shfl_xor_sync(0xffffffffu, pc, o);
    __syncthreads();  // red is reused
    if ((threadIdx.x & 31) == 0) {
        I128Parts q = split(ps);
        red[threadIdx.x >> 5][0] = q.lo;
        red[threadIdx.x >> 5][1] = q.hi;
        red[threadIdx.x >> 5][2] = pc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        i128 s = 0;
        unsigned long long c = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            s += join(red[w][0], red[w][1]);
            c += red[w][2];
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
    uint64_t *table;            // [cap] signature keys
    int64_t cap;                // power of two
    uint32_t *id_a, *id_b;      // signature id per op (radix sort keys)
    uint32_t *ix_a, *ix_b;      // op index (radix sort values)
    unsigned long long *overflow;
};

// Signature -> id = 1 + its slot in the open-addressing table (0 is reserved
// for the sentinel value).  One pass, no id counter: whoever claims or finds
// the slot knows the id.  The pairing only needs "same signature, same id" and
// the stable order inside an id, so the result is deterministic.
__device__ __forceinline__ uint32_t sig_id(const JoinParams &q, uint64_t s, uint64_t h) {
    if (s == EMPTY) return 0;
    const uint64_t mask = (uint64_t)q.cap - 1;
    for (int64_t probe = 0; probe < q.cap; ++probe) {
        uint64_t k = q.table[h];
        if (k == EMPTY) k = atomicCAS((unsigned long long *)&q.table[h], EMPTY, s);
        if (k == EMPTY || k == s) return (uint32_t)h + 1;
        h = (h + 1) & mask;
    }
    atomicAdd(q.overflow, 1ULL);
    return 0;
}

constexpr int ITEMS = 4;  // elements per thread in the streaming kernels (memory-level parallelism)

__global__ void join_hash_kernel(JoinParams q) {
    const int64_t n = q.na + q.nb;
    const uint64_t mask = (uint64_t)q.cap - 1;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * ITEMS;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x * ITEMS + threadIdx.x; base < n; base += stride) {
        uint64_t sg[ITEMS], tk[ITEMS], hh[ITEMS];
#pragma unroll
        for (int u = 0; u < ITEMS; ++u) {
            const int64_t i = base + (int64_t)u * blockDim.x;
            sg[u] = i < n ? __ldcs(i < q.na ? q.sig_a + i : q.sig_b + (i - q.na)) : EMPTY;
        }
        // first probe for all items at once (present signatures resolve here)
#pragma unroll
        for (int u = 0; u < ITEMS; ++u) {
            hh[u] = mix64(sg[u]) & mask;
            tk[u] = q.table[hh[u]];
        }
        uint32_t d[ITEMS];
#pragma unroll
        for (int u = 0; u < ITEMS; ++u) {
            const int64_t i = base + (int64_t)u * blockDim.x;
            d[u] = (i >= n || (tk[u] == sg[u] && sg[u] != EMPTY)) ? (uint32_t)hh[u] + 1
                                                                   : sig_id(q, sg[u], hh[u]);
        }
        __syncwarp();  // reconverge: the stores below must be whole-warp (coalesced) stores
#pragma unroll
        for (int u = 0; u < ITEMS; ++u) {
            const int64_t i = base + (int64_t)u * blockDim.x;
            if (i >= n) continue;
            const bool a = i < q.na;
            const int64_t li = a ? i : i - q.na;
            __stcs((a ? q.id_a : q.id_b) + li, d[u]);
            __stcs((a ? q.ix_a : q.ix_b) + li, (uint32_t)li);
        }
    }
}

// runs of equal ids in a sorted id column -> first[id], end[id]
constexpr int RB_ITEMS = 8;  // consecutive sorted positions per thread (two 16-byte loads)

__global__ void run_bounds_kernel(const uint32_t *sorted, int64_t n, int32_t *first, int32_t *end) {
    const int64_t p0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * RB_ITEMS;
    if (p0 >= n) return;
    uint32_t v[RB_ITEMS + 2];
    v[0] = p0 > 0 ? __ldg(sorted + p0 - 1) : 0xFFFFFFFFu;
    if (p0 + RB_ITEMS <= n && (p0 & 3) == 0) {
        const uint4 a = __ldcs(reinterpret_cast<const uint4 *>(sorted + p0));
        const uint4 b = __ldcs(reinterpret_cast<const uint4 *>(sorted + p0 + 4));
        v[1] = a.x; v[2] = a.y; v[3] = a.z; v[4] = a.w; v[5] = b.x; v[6] = b.y; v[7] = b.z; v[8] = b.w;
    } else {
#pragma unroll
        for (int u = 0; u < RB_ITEMS; ++u) v[u + 1] = p0 + u < n ? __ldg(sorted + p0 + u) : 0xFFFFFFFFu;
    }
    v[RB_ITEMS + 1] = p0 + RB_ITEMS < n ? __ldg(sorted + p0 + RB_ITEMS) : 0xFFFFFFFFu;
#pragma unroll
    for (int u = 0; u < RB_ITEMS; ++u) {
        const int64_t p = p0 + u;
        if (p >= n) break;
        const uint32_t d = v[u + 1];
        if (p == 0 || v[u] != d) first[d] = (int32_t)p;
        if (p == n - 1 || v[u + 2] != d) end[d] = (int32_t)(p + 1);
    }
}

// The pairing in sorted order, written back to A order without a random
// 4-byte scatter over the whole match column (partial-sector writes that miss
// L2 cost a DRAM read-modify-write each).  Pass 1 (sorted order) computes each
// A op's partner and appends (i, j) to the bucket of i >> PAIR_BSH: the
// bucket sizes are known up front (sorted A is a permutation of 0..na-1), so
// bucket b owns stage[b << PAIR_BSH, ...) and a block reserves its share with
// one atomic per bucket.  Pass 2 walks the stage in order and scatters inside
// one bucket's 4 MB window of match_a at a time (L2-resident, full-sector
// write-back).
constexpr int PAIR_BSH = 20;
constexpr int PAIR_THREADS = 256;
constexpr int PAIR_ITEMS = 16;
constexpr int PAIR_MAXB = 2048;  // na < 2^31

__global__ void __launch_bounds__(PAIR_THREADS) join_pair_bucket_kernel(
    const uint32_t *da, const uint32_t *xa, int64_t na, const int32_t *first_a, const uint32_t *xb,
    const int32_t *first_b, const int32_t *end_b, unsigned int *cursor, uint2 *stage) {
    __shared__ int hist[PAIR_MAXB];
    __shared__ int base[PAIR_MAXB];
    const int nbk = (int)((na + (1LL << PAIR_BSH) - 1) >> PAIR_BSH);
    for (int b = threadIdx.x; b < nbk; b += PAIR_THREADS) hist[b] = 0;
    __syncthreads();
    const int64_t p0 = (int64_t)blockIdx.x * PAIR_THREADS * PAIR_ITEMS + threadIdx.x;
    uint32_t i[PAIR_ITEMS];
    int32_t j[PAIR_ITEMS], r[PAIR_ITEMS];
    uint32_t d[PAIR_ITEMS];
#pragma unroll
    for (int u = 0; u < PAIR_ITEMS; ++u) {
        const int64_t p = p0 + (int64_t)u * PAIR_THREADS;
        d[u] = p < na ? __ldcs(da + p) : 0;
        i[u] = p < na ? __ldcs(xa + p) : 0;
    }
#pragma unroll
    for (int u = 0; u < PAIR_ITEMS; ++u) {
        const int64_t p = p0 + (int64_t)u * PAIR_THREADS;
        const int32_t fa = first_a[d[u]], fb = first_b[d[u]], eb = end_b[d[u]];
        const int32_t t = (int32_t)p - fa;
        j[u] = (p < na && eb > 0 && t < eb - fb) ? (int32_t)xb[fb + t] : -1;
    }
#pragma unroll
    for (int u = 0; u < PAIR_ITEMS; ++u) {
        const int64_t p = p0 + (int64_t)u * PAIR_THREADS;
        r[u] = p < na ? atomicAdd(&hist[i[u] >> PAIR_BSH], 1) : 0;
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nbk; b += PAIR_THREADS)
        base[b] = hist[b] ? (int)atomicAdd(cursor + b, (unsigned)hist[b]) : 0;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PAIR_ITEMS; ++u) {
        const int64_t p = p0 + (int64_t)u * PAIR_THREADS;
        if (p >= na) continue;
        const int b = (int)(i[u] >> PAIR_BSH);
        stage[((int64_t)b << PAIR_BSH) + base[b] + r[u]] = make_uint2(i[u], (uint32_t)j[u]);
    }
}

// B operators beyond A's occurrence count of their signature: B-only.  One
// thread per signature id (table slot): the B-only ops of id d are the tail
// [first_b + count_a, end_b) of its run in sorted B (few ids have any).
__global__ void join_bonly_kernel(int64_t D, const uint32_t *xb, const int32_t *first_b, const int32_t *end_b,
                                  const int32_t *first_a, const int32_t *end_a, int32_t *b_only,
                                  unsigned int *n_bonly) {
    const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (d >= D) return;
    const int32_t eb = end_b[d];
    if (eb <= 0) return;
    const int32_t ea = end_a[d];
    const int32_t ca = ea > 0 ? ea - first_a[d] : 0;
    const int32_t fb = first_b[d];
    if (fb + ca >= eb) return;
    const unsigned base = atomicAdd(n_bonly, (unsigned)(eb - fb - ca));  // one reservation per id
    for (int32_t q = fb + ca; q < eb; ++q) b_only[base + (q - fb - ca)] = (int32_t)xb[q];
}

struct JoinSideDev {
    const int64_t *start, *end, *rank;
    const double *joules, *work;
};

__device__ __forceinline__ double div_or_same(double e, const double *work, int64_t i) {
    return work ? __ddiv_rn(e, work[i]) : e;
}

// Pass 1.5 and 2 of the pairing write-back, fused with the A-side findings.
// Pass 1.5 re-partitions every bucket of the stage by window (i >> WIN_BSH,
// 16384 A ops) -- again with known window sizes, so window w owns
// stage2[w << WIN_BSH, ...).  Pass 2 gives each window to one CTA: it lays the
// window's partners out in shared memory, then walks the window's A ops in
// order -- coalesced match_a writes, coalesced A-side reads, the verdict, and
// coalesced finding columns -- with only the B-side reads random.
#ifndef DW_WF_MINB
#define DW_WF_MINB 2
#endif
#ifndef DW_SUB_MINB
#define DW_SUB_MINB 4
#endif
constexpr int WIN_BSH = 14;
constexpr int WIN_OPS = 1 << WIN_BSH;
constexpr int SUB_CHUNK = 4096;  // divides 1 << PAIR_BSH: a chunk never straddles buckets
constexpr int WF_THREADS = 512;

__global__ void __launch_bounds__(256, DW_SUB_MINB) join_pair_sub_kernel(const uint2 *stage, int64_t na, unsigned int *cursor2,
                                                            uint2 *stage2) {
    constexpr int NSUB = 1 << (PAIR_BSH - WIN_BSH);
    __shared__ int hist[NSUB];
    __shared__ int base[NSUB];
    const int64_t c0 = (int64_t)blockIdx.x * SUB_CHUNK;
    const int64_t b = c0 >> PAIR_BSH;
    for (int k = threadIdx.x; k < NSUB; k += 256) hist[k] = 0;
    __syncthreads();
    constexpr int PER = SUB_CHUNK / 256;
    uint2 e[PER];
    int r[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int64_t q = c0 + (int64_t)u * 256 + threadIdx.x;
        e[u] = q < na ? __ldcs(stage + q) : make_uint2(0, 0);
        r[u] = q < na ? atomicAdd(&hist[(e[u].x >> WIN_BSH) & (NSUB - 1)], 1) : 0;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < NSUB; k += 256)
        base[k] = hist[k] ? (int)atomicAdd(cursor2 + (b << (PAIR_BSH - WIN_BSH)) + k, (unsigned)hist[k]) : 0;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int64_t q = c0 + (int64_t)u * 256 + threadIdx.x;
        if (q >= na) continue;
        const int64_t w = e[u].x >> WIN_BSH;
        stage2[(w << WIN_BSH) + base[w & (NSUB - 1)] + r[u]] = e[u];
    }
}

// (join_window_findings: two 512-thread CTAs per SM with one finding per
// thread per step -- the kernel waits on the B-side loads, so warps in
// flight beat unrolled independent loads: U=4 at 1 CTA/SM 1.96 ms, U=2 at 2
// 1.89, U=1 at 2 1.82 ms; U=1 at 3 2.15.  join_pair_sub at 4 CTAs per SM
// instead of 3: 0.71 -> 0.49 ms)
__global__ void __launch_bounds__(WF_THREADS, DW_WF_MINB) join_window_findings_kernel(
    const uint2 *stage2, int64_t na, int32_t *match_a, JoinSideDev A, JoinSideDev B, double threshold, FindCols o,
    double *epw_a, double *epw_b, unsigned long long *n_matched) {
    extern __shared__ int32_t jw[];  // [WIN_OPS]
    const int64_t i0 = (int64_t)blockIdx.x << WIN_BSH;
    const int n = (int)(na - i0 < (int64_t)WIN_OPS ? na - i0 : (int64_t)WIN_OPS);
    for (int q = threadIdx.x; q < n; q += WF_THREADS) {
        const uint2 e = __ldcs(stage2 + i0 + q);
        jw[e.x - (uint32_t)i0] = (int32_t)e.y;
    }
    __syncthreads();
#ifndef DW_WF_U
#define DW_WF_U 1
#endif
    constexpr int U = DW_WF_U;
    unsigned cnt = 0;
    for (int q0 = threadIdx.x; q0 < n; q0 += WF_THREADS * U) {
        int32_t j[U];
        double ea[U], eb[U];
        int64_t la[U], lb[U], tie[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int q = q0 + u * WF_THREADS;
            const int64_t i = i0 + q;
            const bool in = q < n;
            j[u] = in ? jw[q] : -1;
            ea[u] = in ? __ldcs(A.joules + i) : 0.0;
            la[u] = in ? __ldcs(A.end + i) - __ldcs(A.start + i) : 0;
            tie[u] = in && A.rank && o.klo ? __ldcs(A.rank + i) : i;  // only a stored low key needs the rank
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            eb[u] = 0.0;
            lb[u] = 0;
            if (j[u] >= 0) {
                eb[u] = B.joules[j[u]];
                lb[u] = B.end[j[u]] - B.start[j[u]];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int q = q0 + u * WF_THREADS;
            if (q >= n) continue;
            const int64_t i = i0 + q;
            match_a[i] = j[u];
            const Verdict v = judge(ea[u], eb[u], la[u], lb[u], 0.0, threshold);
            const double pa = div_or_same(ea[u], A.work, i);
            const double pb = j[u] >= 0 ? div_or_same(eb[u], B.work, j[u]) : 0.0;
            store_finding(o, i, ea[u], eb[u], la[u], lb[u], v, tie[u], pa, pb);
            if (epw_a) epw_a[i] = pa;
            if (epw_b) epw_b[i] = pb;
            cnt += j[u] >= 0;
        }
    }
    for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(n_matched, (unsigned long long)cnt);
}

__global__ void join_count_kernel(const unsigned long long *matched, int64_t na, int64_t b_only, int64_t *cnt) {
    if (threadIdx.x != 0) return;
    const int64_t m = (int64_t)*matched;
    cnt[0] = na + b_only;
    cnt[1] = m;
    cnt[2] = na - m;
    cnt[3] = b_only;
}

// B-only findings: numbered na + position in B order
__global__ void join_findings_b_kernel(int64_t na, int64_t n_bonly, const int32_t *b_only,
                                       JoinSideDev B, double threshold, FindCols o, double *epw_a,
                                       double *epw_b) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n_bonly) return;
    const int32_t j = b_only[r];
    const int64_t f = na + r;
    const double eb = B.joules[j];
    const int64_t lb = B.end[j] - B.start[j];
    const Verdict v = judge(0.0, eb, 0, lb, 0.0, threshold);
    const double pb = div_or_same(eb, B.work, j);
    store_finding(o, f, 0.0, eb, 0, lb, v, -1, 0.0, pb);  // nodes_a == () sorts first
    if (epw_a) epw_a[f] = 0.0;
    if (epw_b) epw_b[f] = pb;
}

// ---------------------------------------------------- K5' bucketed join (no sort)
// The pairing needs, per signature, its A ops and its B ops in op order; the
// t-th A occurrence pairs with the t-th B occurrence.  Instead of a full radix
// sort by signature id, the ops are partitioned ONCE by signature bucket (a
// range of JB_SPB table slots) with a stable scatter, and one CTA per bucket
// ranks the occurrences of its few hundred signatures in shared memory:
//   jb_hash      per op: table slot of its signature (as K5), plus the per-tile
//                histogram of the bucket id's low 6-bit digit;
//   jb_pass<1>, jb_hist2, jb_pass<2>
//                two stable partition passes (LSD radix, 6-bit digits of the
//                12-bit bucket id), each with its tile x digit count matrix
//                scanned digit-major (jb_colsum / jb_base / jb_apply): the ops
//                end up grouped by bucket, in op order inside a bucket, as
//                (slot << 32 | op index);
//   jb_bounds    each bucket's range (binary search of the grouped column);
//   jb_bucket    per bucket: B's occurrences ranked per slot the same way and
//                laid out by (slot, occurrence); A's occurrences ranked and
//                paired with B's t-th occurrence; the pairs go straight into
//                the A-window stage of K5's findings pass; B ops beyond A's
//                count of their signature set a bit of the B-only bitmap;
//   jb_bonly_*   the bitmap compacted into the B-only list, in B order.
constexpr int JB_NB = 2048;             // signature buckets (+1 for the all-ones signature)
constexpr int JB_NBB = JB_NB + 1;       // bucket ids < 2^12: two 6-bit digits
constexpr int JB_SPB_MAX = 2048;        // table slots per bucket: cap <= JB_NB * JB_SPB_MAX
constexpr int JB_THREADS = 512;         // 16 warps
#ifndef DW_JB_BT
#define DW_JB_BT 512
#endif
constexpr int JB_BT = DW_JB_BT;         // threads of the bucket kernel
constexpr int JB_BW = JB_BT / 32;
constexpr int JB_WARPS = JB_THREADS / 32;
constexpr int JB_DIG = 64;              // radix of the two partition passes
#ifndef DW_JB_T
#define DW_JB_T 4096
#endif
#ifndef DW_JB_PT
#define DW_JB_PT 256
#endif
#ifndef DW_JB_PMINB
#define DW_JB_PMINB 3
#endif
constexpr int JB_T1 = DW_JB_T;          // ops per tile, hash + pass 1
constexpr int JB_T2 = DW_JB_T;          // ops per tile, pass 2 (JB_T1 == JB_T2)
constexpr int JB_PT = DW_JB_PT;         // threads of a partition pass (16 ops per thread)
// measured (C4 passes 1 + 2): 8192-op tiles x 512 threads at 2 CTAs/SM 2.21 ms;
// 4096 x 256 at 4 CTAs 1.93, at 3 (85 registers) 1.70, at 2 2.08; 2048 x 128
// at 8 CTAs 1.84 (+ larger count matrices); 8192 x 1024 2.61
constexpr int JB_PW = JB_PT / 32;
static_assert(JB_T2 % (2 * JB_PT) == 0, "partition pass: an even number of ops per lane");
constexpr int JB_SEG = 256;             // tile segments of a matrix scan

struct JbSide {
    const uint64_t *sig;
    int64_t n;
    uint32_t *slot;            // [n] table slot of each op's signature (cap: the all-ones signature)
    uint32_t *mat1, *mat2;     // [ntile][JB_DIG] digit counts -> output offsets, passes 1 / 2
    uint32_t *part;            // [JB_SEG][JB_DIG] scan scratch
    unsigned long long *tmp;   // [n] after pass 1: (slot << 32 | op index), by low digit
    unsigned long long *scat;  // [n] after pass 2: by bucket, op order kept inside a bucket
    uint32_t *bstart;          // [JB_NBB + 1] first position of each bucket in scat
};

struct JbParams {
    JbSide s[2];
    int64_t nt1[2], nt2[2];    // tiles per side, passes 1 / 2
    uint64_t *table;
    int64_t cap;
    int shift;                 // bucket = slot >> shift
    unsigned long long *overflow;
};

__device__ __forceinline__ uint32_t jb_slot(const JbParams &q, uint64_t s) {
    if (s == EMPTY) return (uint32_t)q.cap;  // its own bucket (JB_NB)
    const uint64_t mask = (uint64_t)q.cap - 1;
    uint64_t h = mix64(s) & mask;
    for (int64_t probe = 0; probe < q.cap; ++probe) {
        uint64_t k = q.table[h];
        if (k == EMPTY) k = atomicCAS((unsigned long long *)&q.table[h], EMPTY, s);
        if (k == EMPTY || k == s) return (uint32_t)h;
        h = (h + 1) & mask;
    }
    atomicAdd(q.overflow, 1ULL);
    return (uint32_t)q.cap;
}

// grid: tiles of side 0 then side 1 (per pass)
__device__ __forceinline__ int jb_side_of(const int64_t *nt, int64_t &t) {
    t = blockIdx.x;
    if (t < nt[0]) return 0;
    t -= nt[0];
    return 1;
}

__global__ void __launch_bounds__(JB_THREADS) jb_hash_kernel(JbParams q) {
    __shared__ unsigned int h[JB_DIG];
    int64_t t;
    const int side = jb_side_of(q.nt1, t);
    const JbSide &S = q.s[side];
    if (threadIdx.x < JB_DIG) h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t i0 = t * JB_T1, i1 = min(i0 + JB_T1, S.n);
    for (int64_t base = i0 + threadIdx.x; base < i1; base += (int64_t)JB_THREADS * ITEMS) {
        uint64_t sg[ITEMS];
#pragma unroll
        for (int u = 0; u < ITEMS; ++u) {
            const int64_t i = base + (int64_t)u * JB_THREADS;
            sg[u] = i < i1 ? __ldcs(S.sig + i) : EMPTY;
        }
#pragma unroll
        for (int u = 0; u < ITEMS; ++u) {
            const int64_t i = base + (int64_t)u * JB_THREADS;
            if (i >= i1) continue;
            const uint32_t sl = jb_slot(q, sg[u]);
            S.slot[i] = sl;
            atomicAdd(&h[(sl >> q.shift) & (JB_DIG - 1)], 1u);
        }
    }
    __syncthreads();
    if (threadIdx.x < JB_DIG) S.mat1[t * JB_DIG + threadIdx.x] = h[threadIdx.x];
}

// Digit-major exclusive scan of a [ntile][JB_DIG] count matrix, in place:
// segment sums, then (one block per side) digit totals, digit bases and
// segment bases, then the segments' running sums.
__global__ void jb_colsum_kernel(JbParams q, int pass) {
    const int side = blockIdx.y;
    const JbSide &S = q.s[side];
    uint32_t *mat = pass == 1 ? S.mat1 : S.mat2;
    const int64_t nt = pass == 1 ? q.nt1[side] : q.nt2[side];
    const int d = threadIdx.x & (JB_DIG - 1);
    const int seg = blockIdx.x * (blockDim.x / JB_DIG) + threadIdx.x / JB_DIG;
    if (seg >= JB_SEG) return;
    const int64_t per = ceil_div(nt, JB_SEG);
    const int64_t t0 = seg * per, t1 = min(t0 + per, nt);
    uint32_t sum = 0;
    for (int64_t t = t0; t < t1; ++t) sum += mat[t * JB_DIG + d];
    S.part[seg * JB_DIG + d] = sum;
}

__global__ void __launch_bounds__(JB_DIG) jb_base_kernel(JbParams q) {
    const JbSide &S = q.s[blockIdx.x];
    const int d = threadIdx.x;  // one thread per digit
    uint32_t tot = 0;
    for (int seg = 0; seg < JB_SEG; ++seg) tot += S.part[seg * JB_DIG + d];
    // exclusive scan of the 64 digit totals (two warps)
    __shared__ uint32_t ws[2];
    const int lane = d & 31, warp = d >> 5;
    uint32_t x = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    uint32_t run = (warp ? ws[0] : 0) + x - tot;
    for (int seg = 0; seg < JB_SEG; ++seg) {
        const uint32_t v = S.part[seg * JB_DIG + d];
        S.part[seg * JB_DIG + d] = run;
        run += v;
    }
}

__global__ void jb_apply_kernel(JbParams q, int pass) {
    const int side = blockIdx.y;
    const JbSide &S = q.s[side];
    uint32_t *mat = pass == 1 ? S.mat1 : S.mat2;
    const int64_t nt = pass == 1 ? q.nt1[side] : q.nt2[side];
    const int d = threadIdx.x & (JB_DIG - 1);
    const int seg = blockIdx.x * (blockDim.x / JB_DIG) + threadIdx.x / JB_DIG;
    if (seg >= JB_SEG) return;
    const int64_t per = ceil_div(nt, JB_SEG);
    const int64_t t0 = seg * per, t1 = min(t0 + per, nt);
    uint32_t run = S.part[seg * JB_DIG + d];
    for (int64_t t = t0; t < t1; ++t) {
        const uint32_t v = mat[t * JB_DIG + d];
        mat[t * JB_DIG + d] = run;
        run += v;
    }
}

// The lanes of a warp step holding the same key (< 2^NB; invalid lanes get
// an empty mask): NB + 1 ballots, or one match.any.  Ballots measured faster
// for both the 6-bit pass digits (C4 passes 1.33 / 1.15 -> 1.11 / 1.08 ms) and
// the 11-bit bucket slots (1.91 -> 1.73 ms).
#ifndef DW_JB_MATCH_PASS
#define DW_JB_MATCH_PASS 0
#endif
#ifndef DW_JB_MATCH_BUCKET
#define DW_JB_MATCH_BUCKET 0
#endif
template <int NB, bool MATCH>
__device__ __forceinline__ unsigned jb_peers(uint32_t key, bool valid) {
    if (MATCH) {
        const unsigned r = __match_any_sync(0xffffffffu, valid ? key : 0xFFFFFFFFu);
        return valid ? r : 0u;
    }
    unsigned r = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const bool on = (key >> b) & 1u;
        const unsigned m = __ballot_sync(0xffffffffu, on);
        r &= on ? m : ~m;
    }
    return valid ? r : 0u;
}

// One stable partition pass by a 6-bit digit of the bucket id (tile of
// JB_T2 ops, 16 per thread).  Each warp owns a contiguous stretch of the
// tile and walks it in op order: every op's rank among the equal digits of
// the stretch (match.any groups, the warp's running counts in shared memory);
// then a scan over the tile (digit-major, warps in order inside a digit); the
// ops are laid out by digit in shared memory and written out in runs
// (coalesced), at the tile's offset of each digit from the scanned count
// matrix.
template <int PASS>
__global__ void __launch_bounds__(JB_PT, DW_JB_PMINB) jb_pass_kernel(JbParams q) {
    constexpr int STEPS = JB_T2 / JB_PT;  // ops per lane
    extern __shared__ __align__(16) unsigned char jb_smem[];
    unsigned long long *lay = reinterpret_cast<unsigned long long *>(jb_smem);  // [JB_T2]
    __shared__ uint32_t cnt[JB_PW][JB_DIG];
    __shared__ uint32_t lstart[JB_DIG], gstart[JB_DIG], half0;
    int64_t t;
    const int side = jb_side_of(q.nt2, t);
    const JbSide &S = q.s[side];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t t0 = t * JB_T2;
    const int nt = (int)min((int64_t)JB_T2, S.n - t0);
    const int64_t w0 = t0 + (int64_t)warp * (STEPS * 32);
    const int dshift = 32 + q.shift + (PASS == 1 ? 0 : 6);
    unsigned long long e[STEPS];  // (slot << 32 | op index)
#pragma unroll
    for (int k = 0; k < STEPS; ++k) {
        const int64_t i = w0 + k * 32 + lane;
        if (PASS == 1)
            e[k] = i < S.n ? ((unsigned long long)__ldcs(S.slot + i) << 32) | (unsigned long long)(uint32_t)i
                           : ~0ULL;
        else
            e[k] = i < S.n ? __ldcs(S.tmp + i) : ~0ULL;
    }
    // each op's rank among the equal digits of this warp's stretch (op order):
    // the lanes holding the same digit in one step (match.any), the group's
    // lowest lane reads and advances the warp's running count of that digit
    cnt[warp][lane] = 0;
    cnt[warp][lane + 32] = 0;
    __syncwarp();
    uint32_t rk[STEPS / 2];  // two 16-bit ranks per register (< STEPS * 32)
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int k = 0; k < STEPS; ++k) {
        const bool valid = e[k] != ~0ULL;
        const uint32_t d = (uint32_t)(e[k] >> dshift) & (JB_DIG - 1);
        const unsigned peers = jb_peers<6, DW_JB_MATCH_PASS>(d, valid);
        const int leader = (__ffs(peers) - 1) & 31;
        uint32_t old = 0;
        if (lane == leader && valid) {
            old = cnt[warp][d];
            cnt[warp][d] = old + __popc(peers);
        }
        const uint32_t r = __shfl_sync(0xffffffffu, old, leader) + __popc(peers & lt);
        if (k & 1) rk[k >> 1] |= r << 16; else rk[k >> 1] = r;
        __syncwarp();
    }
    __syncthreads();
    if (warp < 2) {  // digit d = threadIdx.x: tile total, its start inside the tile (two 32-digit halves)
        const int d = threadIdx.x;
        uint32_t tot = 0;
#pragma unroll
        for (int w = 0; w < JB_PW; ++w) tot += cnt[w][d];
        uint32_t x = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        lstart[d] = x - tot;
        if (d == 31) half0 = x;
        gstart[d] = (PASS == 1 ? S.mat1 : S.mat2)[t * JB_DIG + d];
    }
    __syncthreads();
    if (warp < 2) {  // digit starts, and each warp's base inside its digits
        const int d = threadIdx.x;
        uint32_t run = lstart[d] + (d >= 32 ? half0 : 0);
        lstart[d] = run;
#pragma unroll
        for (int w = 0; w < JB_PW; ++w) {
            const uint32_t c = cnt[w][d];
            cnt[w][d] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < STEPS; ++k) {
        if (e[k] == ~0ULL) continue;
        const uint32_t d = (uint32_t)(e[k] >> dshift) & (JB_DIG - 1);
        lay[cnt[warp][d] + ((rk[k >> 1] >> (k & 1 ? 16 : 0)) & 0xFFFFu)] = e[k];
    }
    __syncthreads();
    unsigned long long *dst = PASS == 1 ? S.tmp : S.scat;
#pragma unroll 4
    for (int x = threadIdx.x; x < nt; x += JB_PT) {  // runs per digit: consecutive threads, consecutive positions
        const unsigned long long v = lay[x];
        const uint32_t d = (uint32_t)(v >> dshift) & (JB_DIG - 1);
        dst[gstart[d] + (x - lstart[d])] = v;
    }
}

// histogram of pass 2's digit over pass 1's output, per pass-2 tile
__global__ void __launch_bounds__(256) jb_hist2_kernel(JbParams q) {
    __shared__ unsigned int h[JB_DIG];
    int64_t t;
    const int side = jb_side_of(q.nt2, t);
    const JbSide &S = q.s[side];
    if (threadIdx.x < JB_DIG) h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t i0 = t * JB_T2, i1 = min(i0 + JB_T2, S.n);
    const int dshift = 32 + q.shift + 6;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += 256)
        atomicAdd(&h[(uint32_t)(__ldcs(S.tmp + i) >> dshift) & (JB_DIG - 1)], 1u);
    __syncthreads();
    if (threadIdx.x < JB_DIG) S.mat2[t * JB_DIG + threadIdx.x] = h[threadIdx.x];
}

// bucket boundaries in the partitioned column (sorted by bucket): one thread per bucket
__global__ void jb_bounds_kernel(JbParams q) {
    const int side = blockIdx.y;
    const JbSide &S = q.s[side];
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > JB_NBB) return;
    int64_t lo = 0, hi = S.n;  // first position with bucket >= b
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((uint32_t)(__ldg(S.scat + mid) >> (32 + q.shift)) < (uint32_t)b) lo = mid + 1; else hi = mid;
    }
    S.bstart[b] = (uint32_t)lo;
}

// A warp's walk of [s0, s1) in order, 32 items per step, JB_PF steps of
// loads issued together (independent loads in flight) before they are used.
constexpr int JB_PF = 8;
template <typename F>
__device__ __forceinline__ void jb_walk(const unsigned long long *src, uint32_t s0, uint32_t s1, F &&f) {
    const int lane = threadIdx.x & 31;
    for (uint32_t c = s0; c < s1; c += 32 * JB_PF) {
        unsigned long long e[JB_PF];
#pragma unroll
        for (int k = 0; k < JB_PF; ++k) {
            const uint32_t x = c + k * 32 + lane;
            e[k] = x < s1 ? __ldcg(src + x) : 0ULL;
        }
#pragma unroll
        for (int k = 0; k < JB_PF; ++k) f(e[k], c + k * 32 + lane < s1);
    }
}

struct JbBucketOut {
    uint32_t *bsorted;           // [nb] B ops laid out by (bucket, slot, occurrence)
    unsigned int *cursor;        // [PAIR_MAXB] A-stage bucket fill
    uint2 *stage;                // A-stage (i, partner) by i >> PAIR_BSH
    uint32_t *bonly_bits;        // [ceil(nb / 32)]
};

// dynamic smem: cw[JB_BW][spb] (u32) + totA, totB, startB [spb] + sbh[PAIR_MAXB]
__global__ void __launch_bounds__(JB_BT) jb_bucket_kernel(JbParams q, JbBucketOut o) {
    extern __shared__ __align__(16) unsigned char jb_smem[];
    const int spb = 1 << q.shift;
    uint32_t *cw = reinterpret_cast<uint32_t *>(jb_smem);
    uint32_t *totA = cw + JB_BW * spb;
    uint32_t *totB = totA + spb;
    uint32_t *startB = totB + spb;
    unsigned int *sbh = startB + spb;
    __shared__ uint32_t wsum[JB_BW];
    const int b = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const JbSide &A = q.s[0], &B = q.s[1];
    const uint32_t a0 = A.bstart[b], a1 = A.bstart[b + 1];
    const uint32_t b0 = B.bstart[b], b1 = B.bstart[b + 1];
    const int nslot = b == JB_NB ? 1 : spb;
    const uint32_t smask = (uint32_t)spb - 1u;
    // this warp's contiguous segment of [lo, hi)
    auto seg = [&](uint32_t lo, uint32_t hi, uint32_t &s0, uint32_t &s1) {
        const uint32_t per = (hi - lo + JB_BW - 1) / JB_BW;
        s0 = min(lo + warp * per, hi);
        s1 = min(s0 + per, hi);
    };
    // per-warp counts of the slots over [lo, hi) -> cross-warp exclusive bases, totals
    auto count_pass = [&](const unsigned long long *src, uint32_t lo, uint32_t hi, uint32_t *tot, bool stage_hist) {
        for (int k = threadIdx.x; k < JB_BW * spb; k += JB_BT) cw[k] = 0;
        if (stage_hist)
            for (int k = threadIdx.x; k < PAIR_MAXB; k += JB_BT) sbh[k] = 0;
        __syncthreads();
        uint32_t s0, s1;
        seg(lo, hi, s0, s1);
        uint32_t *mc = cw + warp * spb;
        jb_walk(src, s0, s1, [&](unsigned long long e, bool valid) {
            if (!valid) return;
            atomicAdd(&mc[(uint32_t)(e >> 32) & smask], 1u);
            if (stage_hist) atomicAdd(&sbh[(uint32_t)e >> PAIR_BSH], 1u);
        });
        __syncthreads();
        for (int s = threadIdx.x; s < nslot; s += JB_BT) {
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < JB_BW; ++w) {
                const uint32_t c = cw[w * spb + s];
                cw[w * spb + s] = run;
                run += c;
            }
            tot[s] = run;
        }
        __syncthreads();
    };
    // ---- B: occurrences by slot, laid out at bsorted[b0 + startB[s] + occ]
    count_pass(B.scat, b0, b1, totB, false);
    {  // startB = exclusive scan of totB over the slots
        uint32_t carry = 0;
        for (int c = 0; c < nslot; c += JB_BT) {
            const int s = c + threadIdx.x;
            const uint32_t v = s < nslot ? totB[s] : 0;
            uint32_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) wsum[warp] = x;
            __syncthreads();
            uint32_t wb = 0, all = 0;
#pragma unroll
            for (int w = 0; w < JB_BW; ++w) {
                const uint32_t ws = wsum[w];
                if (w < warp) wb += ws;
                all += ws;
            }
            if (s < nslot) startB[s] = carry + wb + x - v;
            carry += all;
            __syncthreads();
        }
    }
    {
        uint32_t s0, s1;
        seg(b0, b1, s0, s1);
        uint32_t *mc = cw + warp * spb;
        jb_walk(B.scat, s0, s1, [&](unsigned long long e, bool valid) {
            const uint32_t sl = (uint32_t)(e >> 32) & smask;
            const unsigned peers = jb_peers<11, DW_JB_MATCH_BUCKET>(sl, valid);
            const int below = __popc(peers & ((1u << lane) - 1u));
            const uint32_t occ = valid ? mc[sl] + below : 0;
            __syncwarp();
            if (valid && below == 0) mc[sl] += __popc(peers);
            __syncwarp();
            if (valid) o.bsorted[b0 + startB[sl] + occ] = (uint32_t)e;
        });
    }
    __syncthreads();  // bsorted of this bucket complete (block-visible)
    // ---- A: occurrences by slot, paired with B's t-th occurrence
    count_pass(A.scat, a0, a1, totA, true);
    for (int k = threadIdx.x; k < PAIR_MAXB; k += JB_BT)  // reserve this bucket's A-stage ranges
        if (sbh[k]) sbh[k] = atomicAdd(o.cursor + k, sbh[k]);
    for (int s = threadIdx.x; s < nslot; s += JB_BT) {  // B occurrences beyond A's count: B-only
        for (uint32_t t = totA[s]; t < totB[s]; ++t) {
            const uint32_t j = o.bsorted[b0 + startB[s] + t];
            atomicOr(o.bonly_bits + (j >> 5), 1u << (j & 31));
        }
    }
    __syncthreads();
    {
        uint32_t s0, s1;
        seg(a0, a1, s0, s1);
        uint32_t *mc = cw + warp * spb;
        jb_walk(A.scat, s0, s1, [&](unsigned long long e, bool valid) {
            const uint32_t sl = (uint32_t)(e >> 32) & smask, i = (uint32_t)e;
            const unsigned peers = jb_peers<11, DW_JB_MATCH_BUCKET>(sl, valid);
            const int below = __popc(peers & ((1u << lane) - 1u));
            const uint32_t occ = valid ? mc[sl] + below : 0;
            __syncwarp();
            if (valid && below == 0) mc[sl] += __popc(peers);
            __syncwarp();
            if (valid) {
                const int32_t j = occ < totB[sl] ? (int32_t)o.bsorted[b0 + startB[sl] + occ] : -1;
                const unsigned pos = atomicAdd(&sbh[i >> PAIR_BSH], 1u);
                o.stage[((int64_t)(i >> PAIR_BSH) << PAIR_BSH) + pos] = make_uint2(i, (uint32_t)j);
            }
        });
    }
}

// B-only list from the bitmap, in B order: per-block popcounts, their scan, writes
constexpr int BO_WORDS = 2048;  // bitmap words per block (8 per thread)
__global__ void __launch_bounds__(256) bonly_count_kernel(const uint32_t *bits, int64_t nw, uint32_t *bsum) {
    uint32_t c = 0;
    const int64_t w0 = (int64_t)blockIdx.x * BO_WORDS;
    for (int k = threadIdx.x; k < BO_WORDS; k += 256) c += w0 + k < nw ? __popc(bits[w0 + k]) : 0;
    c = __reduce_add_sync(0xffffffffu, c);
    __shared__ uint32_t s[8];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < 8; ++w) t += s[w];
        bsum[blockIdx.x] = t;
    }
}
__global__ void __launch_bounds__(1024) bonly_scan_kernel(uint32_t *bsum, int64_t nblk, unsigned int *total) {
    __shared__ uint32_t carry;
    __shared__ uint32_t ws[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t c = 0; c < nblk; c += 1024) {
        const int64_t k = c + threadIdx.x;
        const uint32_t v = k < nblk ? bsum[k] : 0;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) ws[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = ws[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            ws[lane] = w;
        }
        __syncthreads();
        if (k < nblk) bsum[k] = carry + (warp ? ws[warp - 1] : 0) + x - v;
        __syncthreads();
        if (threadIdx.x == 0) carry += ws[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}
__global__ void __launch_bounds__(256) bonly_write_kernel(const uint32_t *bits, int64_t nw, const uint32_t *bsum,
                                                          int32_t *out) {
    // each thread owns 8 consecutive words; thread order = word order
    const int64_t w0 = (int64_t)blockIdx.x * BO_WORDS + threadIdx.x * 8;
    uint32_t wv[8];
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        wv[k] = w0 + k < nw ? bits[w0 + k] : 0u;
        c += __popc(wv[k]);
    }
    __shared__ uint32_t ws[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    uint32_t base = bsum[blockIdx.x] + x - c;
    for (int w = 0; w < warp; ++w) base += ws[w];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        uint32_t m = wv[k];
        while (m) {
            const int bit = __ffs(m) - 1;
            m &= m - 1;
            out[base++] = (int32_t)(((w0 + k) << 5) + bit);
        }
    }
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
        partials, done, seg, seg_bytes, cub, cub_bytes, total;
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
    L.seg_bytes = dw_rank_segmented_workspace_size(1, std::min<int64_t>(k, 8192));
    L.seg = off; off += au(L.seg_bytes);
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

static int rank_impl(int64_t P, const uint64_t *khi, const uint64_t *klo, const int64_t *tie_rank,
                     int64_t n_a, int64_t k, int64_t *order, double *summary, void *ws,
                     size_t ws_bytes, cudaStream_t s) {
    if (P < 0 || k < 0 || k > P || (P && !khi) || (k && !order) || !ws) return DW_E_ARG;
    RankLayout L = rank_layout(P, k);
    if (ws_bytes < L.total) return DW_E_WORKSPACE;
    char *base = (char *)ws;
    trace_mark(s, "rank:start");
    // the first digit's histogram comes with the waste sum (one read of the keys)
    const bool fused_hist = summary && P > 0 && k > 0;
    if (fused_hist) cudaMemsetAsync(base + L.hist, 0, 4 * HIST_BINS, s);
    if (summary) {
        cudaMemsetAsync(base + L.done, 0, 16, s);
        if (P > 0) {
            static int per_sm = 0;  // one resident wave (no tail), at most 1024 partials
            if (!per_sm && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, waste_sum_kernel, 256, 0) !=
                               cudaSuccess)
                per_sm = 1;
            const int64_t wgrid = std::min<int64_t>(std::min<int64_t>(1024, (int64_t)num_sms() * per_sm),
                                                    blocks_for(P));
            waste_sum_kernel<<<(unsigned)wgrid, 256, 0, s>>>(
                khi, P, (unsigned long long *)(base + L.partials), (unsigned int *)(base + L.done),
                summary, fused_hist ? (unsigned int *)(base + L.hist) : nullptr);
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
    r.tie_rank = tie_rank;
    r.n_a = n_a;
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
        if (!(fused_hist && pos == 128 - HIST_BITS)) {
            cudaMemsetAsync(r.hist, 0, 4 * HIST_BINS, s);
            rank_hist_kernel<<<grid, 512, 0, s>>>(r);
            count_launch();
        }
        rank_select_kernel<<<1, 32, 0, s>>>(r, need);
        count_launch();
        trace_mark(s, "rank:digit");
        unsigned long long sel[3];
        cudaMemcpyAsync(sel, r.sel, sizeof(sel), cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) return DW_E_CUDA;
        const unsigned long long in_bin = sel[2];
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
    trace_mark(s, "rank:compact");
    if (k <= 8192) {
        // the k best of the candidates: the segmented top-k on the candidate
        // keys (a few small radix passes, then a shared-memory bitonic sort --
        // no library sort), mapped back to finding indices
        dw_rank_segment_t seg{r.cand_hi, r.cand_lo, nullptr, 0, (int64_t)nc};
        int64_t *pos = (int64_t *)(base + L.tmp_idx2);
        const int rc = dw_rank_segmented(&seg, 1, k, pos, nullptr, base + L.seg, L.seg_bytes, s);
        if (rc != DW_OK) return rc;
        gather_i64_kernel<<<blocks_for(k), 256, 0, s>>>(r.cand_idx, pos, k, order);
        count_launch();
    } else {
        sort_candidates(base, L, (int64_t)nc, s);
        cudaMemcpyAsync(order, base + L.tmp_idx, 8 * k, cudaMemcpyDeviceToDevice, s);
    }
    trace_mark(s, "rank:sort");
    DW_CHECK_LAUNCH();
    return DW_OK;
}

struct JoinLayout {
    size_t table, counters, id_a, id_b, ix_a, ix_b, sid_a, sid_b, six_a, six_b, first_a, end_a,
        first_b, end_b,
        bonly_tmp, pair_stage, pair_cursor, win_stage, win_cursor, cub, cub_bytes, total;
    // bucketed join (jb): tile x bucket matrices, segment sums, bucket starts,
    // scattered ops, B by (slot, occurrence), B-only bitmap and block sums
    size_t mat_a, mat_b, mat2_a, mat2_b, part_a, part_b, bst_a, bst_b, tmp_a, tmp_b, scat_a, scat_b, bsorted,
        bbits, bsum;
    int64_t cap, D, nt1_a, nt1_b, nt2_a, nt2_b, nw, nblk;
    bool jb;
};

static int64_t pow2_at_least(int64_t x) {
    int64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

// The bucketed join handles tables of up to JB_NB * JB_SPB_MAX slots (2M
// distinct signatures); larger ones take the sort-based path.
static JoinLayout join_layout(int64_t na, int64_t nb, int64_t max_distinct) {
    JoinLayout L{};
    if (max_distinct <= 0 || max_distinct > na + nb) max_distinct = na + nb;
    L.cap = pow2_at_least(std::max<int64_t>(4096, 2 * max_distinct));
    L.jb = L.cap <= (int64_t)JB_NB * JB_SPB_MAX;
    L.D = L.cap + 2;  // ids are table slots + 1; 0 reserved
    size_t off = 0;
    L.table = off; off += au(8 * L.cap);
    L.counters = off; off += au(64);
    L.id_a = off; off += au(4 * na);
    L.id_b = off; off += au(4 * nb);
    L.bonly_tmp = off; off += au(4 * std::max<int64_t>(nb, 1));
    L.pair_stage = off; off += au(8 * std::max<int64_t>(na, 1));
    L.pair_cursor = off; off += au(4 * PAIR_MAXB);
    L.win_stage = off; off += au(8 * std::max<int64_t>(na, 1));
    L.win_cursor = off; off += au(4 * ((std::max<int64_t>(na, 1) + WIN_OPS - 1) / WIN_OPS));
    if (L.jb) {
        L.nt1_a = ceil_div(na, JB_T1);
        L.nt1_b = ceil_div(nb, JB_T1);
        L.nt2_a = ceil_div(na, JB_T2);
        L.nt2_b = ceil_div(nb, JB_T2);
        L.mat_a = off; off += au(4 * JB_DIG * L.nt1_a);
        L.mat_b = off; off += au(4 * JB_DIG * L.nt1_b);
        L.mat2_a = off; off += au(4 * JB_DIG * L.nt2_a);
        L.mat2_b = off; off += au(4 * JB_DIG * L.nt2_b);
        L.part_a = off; off += au(4 * JB_SEG * JB_DIG);
        L.part_b = off; off += au(4 * JB_SEG * JB_DIG);
        L.bst_a = off; off += au(4 * (JB_NBB + 1));
        L.bst_b = off; off += au(4 * (JB_NBB + 1));
        L.tmp_a = off; off += au(8 * na);
        L.tmp_b = off; off += au(8 * nb);
        L.scat_a = off; off += au(8 * na);
        L.scat_b = off; off += au(8 * nb);
        L.bsorted = off; off += au(4 * nb);
        L.nw = ceil_div(std::max<int64_t>(nb, 1), 32);
        L.nblk = ceil_div(L.nw, BO_WORDS);
        L.bbits = off; off += au(4 * L.nw);
        L.bsum = off; off += au(4 * L.nblk);
        L.total = off;
        return L;
    }
    L.ix_a = off; off += au(4 * na);
    L.ix_b = off; off += au(4 * nb);
    L.sid_a = off; off += au(4 * na);
    L.sid_b = off; off += au(4 * nb);
    L.six_a = off; off += au(4 * na);
    L.six_b = off; off += au(4 * nb);
    L.first_a = off; off += au(4 * L.D);
    L.end_a = off; off += au(4 * L.D);
    L.first_b = off; off += au(4 * L.D);
    L.end_b = off; off += au(4 * L.D);
    size_t c1 = 0, c2 = 0;
    const int64_t nmax = std::max<int64_t>(std::max(na, nb), 1);
    cub::DeviceRadixSort::SortPairs(nullptr, c1, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (const uint32_t *)nullptr, (uint32_t *)nullptr, (int)nmax);
    cub::DeviceRadixSort::SortKeys(nullptr, c2, (const int32_t *)nullptr, (int32_t *)nullptr,
                                   (int)std::max<int64_t>(nb, 1));
    L.cub = off;
    L.cub_bytes = std::max(c1, c2);
    off += au(L.cub_bytes);
    L.total = off;
    return L;
}

static int log2_exact(int64_t x) {
    int b = 0;
    while (((int64_t)1 << b) < x) ++b;
    return b;
}

// phase 1 of the bucketed join: pairs into the A stage (by i >> PAIR_BSH), the
// B-only list; returns the B-only count through *n_bonly (host)
static int jb_pairing(const dw_join_side_t *a, const dw_join_side_t *b, const JoinLayout &L, char *base,
                      int32_t *d_b_only, int64_t *n_bonly, cudaStream_t s) {
    const int64_t na = a->n, nb = b->n;
    unsigned long long *counters = (unsigned long long *)(base + L.counters);
    JbParams q{};
    q.table = (uint64_t *)(base + L.table);
    q.cap = L.cap;
    q.shift = log2_exact(L.cap / JB_NB);
    q.overflow = counters;
    const int64_t n2[2] = {na, nb};
    const uint64_t *sig[2] = {a->d_sig, b->d_sig};
    const size_t slot_off[2] = {L.id_a, L.id_b}, mat[2] = {L.mat_a, L.mat_b}, mat2[2] = {L.mat2_a, L.mat2_b},
                 part[2] = {L.part_a, L.part_b}, bst[2] = {L.bst_a, L.bst_b}, tmp[2] = {L.tmp_a, L.tmp_b},
                 scat[2] = {L.scat_a, L.scat_b};
    q.nt1[0] = L.nt1_a;
    q.nt1[1] = L.nt1_b;
    q.nt2[0] = L.nt2_a;
    q.nt2[1] = L.nt2_b;
    for (int k = 0; k < 2; ++k) {
        q.s[k].sig = sig[k];
        q.s[k].n = n2[k];
        q.s[k].slot = (uint32_t *)(base + slot_off[k]);
        q.s[k].mat1 = (uint32_t *)(base + mat[k]);
        q.s[k].mat2 = (uint32_t *)(base + mat2[k]);
        q.s[k].part = (uint32_t *)(base + part[k]);
        q.s[k].bstart = (uint32_t *)(base + bst[k]);
        q.s[k].tmp = (unsigned long long *)(base + tmp[k]);
        q.s[k].scat = (unsigned long long *)(base + scat[k]);
    }
    trace_mark(s, "join:start");
    cudaMemsetAsync(counters, 0, 64, s);
    cudaMemsetAsync(q.table, 0xFF, 8 * L.cap, s);
    const unsigned tiles1 = (unsigned)(L.nt1_a + L.nt1_b), tiles2 = (unsigned)(L.nt2_a + L.nt2_b);
    const dim3 sg(JB_SEG * JB_DIG / 256, 2);
    cudaFuncSetAttribute(jb_pass_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * JB_T2);
    cudaFuncSetAttribute(jb_pass_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * JB_T2);
    if (tiles1) {
        jb_hash_kernel<<<tiles1, JB_THREADS, 0, s>>>(q);
        jb_colsum_kernel<<<sg, 256, 0, s>>>(q, 1);
        jb_base_kernel<<<2, JB_DIG, 0, s>>>(q);
        jb_apply_kernel<<<sg, 256, 0, s>>>(q, 1);
        jb_pass_kernel<1><<<tiles1, JB_PT, 8 * JB_T2, s>>>(q);
        jb_hist2_kernel<<<tiles2, 256, 0, s>>>(q);
        jb_colsum_kernel<<<sg, 256, 0, s>>>(q, 2);
        jb_base_kernel<<<2, JB_DIG, 0, s>>>(q);
        jb_apply_kernel<<<sg, 256, 0, s>>>(q, 2);
        jb_pass_kernel<2><<<tiles2, JB_PT, 8 * JB_T2, s>>>(q);
        count_launch(10);
    }
    jb_bounds_kernel<<<dim3((JB_NBB + 1 + 255) / 256, 2), 256, 0, s>>>(q);
    count_launch();
    trace_mark(s, "join:partition");
    JbBucketOut o{};
    o.bsorted = (uint32_t *)(base + L.bsorted);
    o.cursor = (unsigned int *)(base + L.pair_cursor);
    o.stage = (uint2 *)(base + L.pair_stage);
    o.bonly_bits = (uint32_t *)(base + L.bbits);
    cudaMemsetAsync(o.cursor, 0, 4 * PAIR_MAXB, s);
    cudaMemsetAsync(o.bonly_bits, 0, 4 * L.nw, s);
    const int spb = 1 << q.shift;
    const size_t smem_b = 4 * ((size_t)(JB_BW + 3) * spb + PAIR_MAXB);
    cudaFuncSetAttribute(jb_bucket_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_b);
    jb_bucket_kernel<<<JB_NBB, JB_BT, smem_b, s>>>(q, o);
    count_launch();
    trace_mark(s, "join:bucket");
    if (na) {
        unsigned int *cursor2 = (unsigned int *)(base + L.win_cursor);
        uint2 *stage2 = (uint2 *)(base + L.win_stage);
        const int64_t nwin = (na + WIN_OPS - 1) / WIN_OPS;
        cudaMemsetAsync(cursor2, 0, 4 * nwin, s);
        join_pair_sub_kernel<<<(unsigned)((na + SUB_CHUNK - 1) / SUB_CHUNK), 256, 0, s>>>(o.stage, na, cursor2,
                                                                                           stage2);
        count_launch();
        trace_mark(s, "join:pair_sub");
    }
    unsigned int *n_bo = (unsigned int *)(counters + 3);
    if (nb) {
        uint32_t *bsum = (uint32_t *)(base + L.bsum);
        bonly_count_kernel<<<(unsigned)L.nblk, 256, 0, s>>>(o.bonly_bits, L.nw, bsum);
        bonly_scan_kernel<<<1, 1024, 0, s>>>(bsum, L.nblk, n_bo);
        bonly_write_kernel<<<(unsigned)L.nblk, 256, 0, s>>>(o.bonly_bits, L.nw, bsum, d_b_only);
        count_launch(3);
        trace_mark(s, "join:bonly");
    }
    unsigned long long hc[4] = {0, 0, 0, 0};  // overflow, matched, -, n_bonly
    cudaMemcpyAsync(hc, counters, sizeof(hc), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return DW_E_CUDA;
    if (hc[0]) return DW_E_WORKSPACE;  // more distinct signatures than the table holds
    *n_bonly = (int64_t)(unsigned int)hc[3];
    return DW_OK;
}

static int bits_for(int64_t D) {
    int b = 1;
    while (((int64_t)1 << b) <= D) ++b;
    return b;
}


// ------------------------------------------------ K6s segmented top-k
// The report order of many finding sets at once (one segment per trace pair
// of a corpus): every launch covers all segments (grid.y =
// segment), each with its own radix-select state, so a corpus of S pairs takes
// the same few launches as one pair.  Per segment: the exact waste sum, the
// threshold digit by digit until the keys above it fit SEG_SORT_MAX, their
// compaction, and a bitonic sort in shared memory (no library sort).
constexpr int SEG_SORT_MAX = 8192;   // candidates per segment (24 B each in shared memory)
constexpr int SEG_SORT_THREADS = 1024;
constexpr int SEG_BLOCK = 512;

struct SegDesc {
    const uint64_t *khi, *klo;
    const int64_t *tie_rank;
    int64_t n_a, P, k;
};

struct SegState {
    uint64_t phi, plo, mhi, mlo, thr_hi, thr_lo;
    int64_t need;
    int32_t pos, done;
};

__device__ __forceinline__ uint64_t seg_lo(const SegDesc &d, int64_t i) {
    if (d.klo) return d.klo[i];
    const int64_t tie = i < d.n_a ? (d.tie_rank ? d.tie_rank[i] : i) : -1;
    return key_lo(tie, i);
}

__global__ void seg_init_kernel(const SegDesc *segs, int nseg, SegState *st, unsigned *hist, unsigned *cand_n,
                                unsigned *pending) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s == 0) *pending = 0;
    if (s >= nseg) return;
    SegState z{};
    z.need = segs[s].k;
    z.pos = 128 - HIST_BITS;
    z.done = segs[s].k == 0;  // nothing to rank
    st[s] = z;
    cand_n[s] = 0;
    for (int b = 0; b < HIST_BINS; ++b) hist[s * HIST_BINS + b] = 0;
}

// exact n_waste and wasted sum per segment: block partials, then one block per segment
__global__ void __launch_bounds__(256) seg_waste_kernel(const SegDesc *segs, unsigned long long *partials) {
    const int s = blockIdx.y;
    const SegDesc d = segs[s];
    i128 acc = 0;
    unsigned long long cnt = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.P; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = d.khi[i];
        if (k >> 63) {
            acc += fx_joules(__longlong_as_double((long long)(k & 0x7FFFFFFFFFFFFFFFULL)));
            ++cnt;
        }
    }
    acc = warp_sum_i128(acc);
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    __shared__ unsigned long long red[8][3];
    if ((threadIdx.x & 31) == 0) {
        const I128Parts q = split(acc);
        red[threadIdx.x >> 5][0] = q.lo;
        red[threadIdx.x >> 5][1] = q.hi;
        red[threadIdx.x >> 5][2] = cnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        i128 t = 0;
        unsigned long long c = 0;
        for (int w = 0; w < 8; ++w) {
            t += join(red[w][0], red[w][1]);
            c += red[w][2];
        }
        const I128Parts q = split(t);
        unsigned long long *o = partials + 3 * ((int64_t)s * gridDim.x + blockIdx.x);
        o[0] = q.lo;
        o[1] = q.hi;
        o[2] = c;
    }
}

__global__ void seg_waste_final_kernel(const SegDesc *segs, const unsigned long long *partials, int nblk,
                                       double *summary) {
    const int s = blockIdx.x;
    if (threadIdx.x != 0) return;
    i128 t = 0;
    unsigned long long c = 0;
    for (int b = 0; b < nblk; ++b) {
        const unsigned long long *o = partials + 3 * ((int64_t)s * nblk + b);
        t += join(o[0], o[1]);
        c += o[2];
    }
    summary[4 * s + 0] = (double)c;
    summary[4 * s + 1] = fx_to_double(t, FX_JOULE_BITS);
    summary[4 * s + 2] = (double)segs[s].P;
    summary[4 * s + 3] = 0.0;
}

__global__ void __launch_bounds__(SEG_BLOCK) seg_hist_kernel(const SegDesc *segs, const SegState *st,
                                                              unsigned *hist) {
    const int s = blockIdx.y;
    const SegState g = st[s];
    if (g.done) return;
    const SegDesc d = segs[s];
    __shared__ unsigned h[HIST_BINS];
    for (int b = threadIdx.x; b < HIST_BINS; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const bool need_lo = g.pos < 64 || g.mlo;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.P; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t hi = d.khi[i];
        if ((hi & g.mhi) != g.phi) continue;
        const uint64_t lo = need_lo ? seg_lo(d, i) : 0;
        if ((lo & g.mlo) != g.plo) continue;
        atomicAdd(&h[digit128(hi, lo, g.pos)], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < HIST_BINS; b += blockDim.x)
        if (h[b]) atomicAdd(&hist[s * HIST_BINS + b], h[b]);
}

// one warp per segment: the bin holding the need-th largest key; either the
// keys >= the threshold fit the candidate buffer (done) or the next digit
__global__ void seg_select_kernel(const SegDesc *segs, SegState *st, unsigned *hist, int64_t cap,
                                  unsigned *pending) {
    const int s = blockIdx.x;
    SegState g = st[s];
    if (g.done) return;
    unsigned *h = hist + s * HIST_BINS;
    if (threadIdx.x == 0) {
        int64_t above = 0;
        int b = HIST_BINS - 1;
        for (; b > 0; --b) {
            if (above + (int64_t)h[b] >= g.need) break;
            above += h[b];
        }
        const uint64_t dig = (uint64_t)b;
        if (g.pos >= 64) {
            g.thr_hi = g.phi | (dig << (g.pos - 64));
            g.thr_lo = 0;
        } else {
            g.thr_hi = g.phi;
            g.thr_lo = g.plo | (dig << g.pos);
        }
        // keys >= the threshold: those above the prefix (counted in earlier
        // digits), the bins above b, and bin b
        const int64_t cand = (segs[s].k - g.need) + above + (int64_t)h[b];
        if (g.pos == 0 || cand <= cap) {
            g.done = 1;
        } else {
            g.need -= above;
            g.phi = g.thr_hi;
            g.plo = g.thr_lo;
            if (g.pos >= 64) g.mhi |= ((uint64_t)(HIST_BINS - 1)) << (g.pos - 64);
            else g.mlo |= ((uint64_t)(HIST_BINS - 1)) << g.pos;
            g.pos -= HIST_BITS;
            atomicAdd(pending, 1u);
        }
        st[s] = g;
    }
    __syncwarp();
    for (int b = threadIdx.x; b < HIST_BINS; b += 32) h[b] = 0;
}

__global__ void __launch_bounds__(256) seg_compact_kernel(const SegDesc *segs, const SegState *st, int64_t cap,
                                                          uint64_t *chi, uint64_t *clo, int64_t *cidx,
                                                          unsigned *cand_n) {
    const int s = blockIdx.y;
    const SegDesc d = segs[s];
    if (d.k == 0) return;
    const uint64_t th = st[s].thr_hi, tl = st[s].thr_lo;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.P; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t hi = d.khi[i];
        if (hi < th) continue;
        const uint64_t lo = seg_lo(d, i);
        if (hi == th && lo < tl) continue;
        const unsigned slot = atomicAdd(&cand_n[s], 1u);
        if ((int64_t)slot < cap) {
            const int64_t o = (int64_t)s * cap + slot;
            chi[o] = hi;
            clo[o] = lo;
            cidx[o] = i;
        }
    }
}

// one CTA per segment: bitonic sort of the candidates, descending (hi, lo)
// (keys are distinct: lo carries the finding index), best k indices out
__global__ void __launch_bounds__(SEG_SORT_THREADS) seg_sort_kernel(const SegDesc *segs, int64_t cap,
                                                                    const uint64_t *chi, const uint64_t *clo,
                                                                    const int64_t *cidx, const unsigned *cand_n,
                                                                    int64_t k, int64_t *order, int *overflow) {
    extern __shared__ __align__(16) unsigned char seg_smem[];
    const int s = blockIdx.x;
    int n = (int)min((int64_t)cand_n[s], cap);
    if ((int64_t)cand_n[s] > cap && threadIdx.x == 0) atomicOr(overflow, 1);
    int m = 1;
    while (m < n) m <<= 1;
    uint64_t *sh = reinterpret_cast<uint64_t *>(seg_smem);
    uint64_t *sl = sh + m;
    int64_t *si = reinterpret_cast<int64_t *>(sl + m);
    for (int x = threadIdx.x; x < m; x += blockDim.x) {
        const bool in = x < n;
        const int64_t o = (int64_t)s * cap + x;
        sh[x] = in ? chi[o] : 0;
        sl[x] = in ? clo[o] : 0;
        si[x] = in ? cidx[o] : -1;
    }
    __syncthreads();
    for (int size = 2; size <= m; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int x = threadIdx.x; x < m; x += blockDim.x) {
                const int y = x ^ stride;
                if (y > x) {
                    const bool desc = (x & size) == 0;  // descending runs first: the whole array ends descending
                    const bool less = sh[x] < sh[y] || (sh[x] == sh[y] && sl[x] < sl[y]);
                    if (less == desc) {
                        const uint64_t th = sh[x], tl = sl[x];
                        const int64_t ti = si[x];
                        sh[x] = sh[y]; sl[x] = sl[y]; si[x] = si[y];
                        sh[y] = th; sl[y] = tl; si[y] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
    const int64_t ks = segs[s].k;
    for (int64_t x = threadIdx.x; x < k; x += blockDim.x) order[(int64_t)s * k + x] = x < ks && x < n ? si[x] : -1;
}


// The top-k rows of a join for the host report, in one launch: per row r of
// the report order, its A / B operators (join numbering: f < n_a is A op f
// with partner match_a[f]; else the B-only op b_only[f - n_a]), their joules
// and latencies.  out[6][k] (int64; joules as their f64 bits): ia, ib, la,
// lb, ea, eb -- one device->host copy instead of a dozen gathers.
__global__ void topk_rows_kernel(const int64_t *order, int64_t k, int64_t n_a, const int32_t *match_a,
                                 const int32_t *b_only, const double *ja, const double *jb, const int64_t *sa,
                                 const int64_t *ea, const int64_t *sb, const int64_t *eb, int64_t *out) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= k) return;
    const int64_t f = order[r];
    int64_t ia = -1, ib = -1;
    if (f >= 0 && f < n_a) {
        ia = f;
        ib = match_a[f];
    } else if (f >= n_a) {
        ib = b_only[f - n_a];
    }
    out[r] = ia;
    out[k + r] = ib;
    out[2 * k + r] = ia >= 0 ? ea[ia] - sa[ia] : 0;
    out[3 * k + r] = ib >= 0 ? eb[ib] - sb[ib] : 0;
    out[4 * k + r] = __double_as_longlong(ia >= 0 ? ja[ia] : 0.0);
    out[5 * k + r] = __double_as_longlong(ib >= 0 ? jb[ib] : 0.0);
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
    return rank_impl(P, f->d_key_hi, f->d_key_lo, f->d_tie_rank, f->n_a, k, d_order, d_summary,
                     d_workspace, workspace_bytes, (cudaStream_t)stream);
}

size_t dw_join_workspace_size(int64_t na, int64_t nb, int64_t max_distinct) {
    return join_layout(na, nb, max_distinct).total;
}

// phase 1: pairing only (signatures; no joules needed) -> stage2, b_only,
// *n_bonly_out; phase 2: the findings (joules); 3: both
static int join_impl(const dw_join_side_t *a, const dw_join_side_t *b, int64_t max_distinct, double threshold,
                     dw_findings_t *out, int32_t *d_match_a, int32_t *d_b_only, double *d_epw_a, double *d_epw_b,
                     int64_t *d_count, void *d_workspace, size_t workspace_bytes, dw_stream_t stream, int phase,
                     int64_t *n_bonly_io) {
    if (!a || !b || !d_workspace) return DW_E_ARG;
    if ((phase & 2) && (!(threshold > 0.0 && threshold <= 1.0))) return DW_E_ARG;
    if ((phase & 2) && (!out || !out->d_key_hi || !d_count)) return DW_E_ARG;
    const int64_t na = a->n, nb = b->n;
    if (na < 0 || nb < 0 || na + nb >= ((int64_t)1 << 31)) return DW_E_ARG;
    if ((na && (!a->d_sig || !a->d_start || !a->d_end || !d_match_a)) ||
        (nb && (!b->d_sig || !b->d_start || !b->d_end || !d_b_only)))
        return DW_E_ARG;
    if ((phase & 2) && ((na && !a->d_joules) || (nb && !b->d_joules))) return DW_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    JoinLayout L = join_layout(na, nb, max_distinct);
    if (workspace_bytes < L.total) return DW_E_WORKSPACE;
    char *base = (char *)d_workspace;
    unsigned long long *counters = (unsigned long long *)(base + L.counters);
    int64_t b_only = 0;
    if ((phase & 1) && L.jb) {
        const int rc = jb_pairing(a, b, L, base, d_b_only, &b_only, s);
        if (rc != DW_OK) return rc;
        if (n_bonly_io) *n_bonly_io = b_only;
    } else if (phase & 1) {
        JoinParams q{};
        q.sig_a = a->d_sig;
        q.sig_b = b->d_sig;
        q.na = na;
        q.nb = nb;
        q.table = (uint64_t *)(base + L.table);
        q.cap = L.cap;
        q.id_a = (uint32_t *)(base + L.id_a);
        q.id_b = (uint32_t *)(base + L.id_b);
        q.ix_a = (uint32_t *)(base + L.ix_a);
        q.ix_b = (uint32_t *)(base + L.ix_b);
        // counters: [0] overflow, [1] matched, [2] next_id (u32), [3] n_bonly (u32)
        q.overflow = counters;
        unsigned int *n_bonly = (unsigned int *)(counters + 3);
        trace_mark(s, "join:start");
        cudaMemsetAsync(counters, 0, 64, s);
        cudaMemsetAsync(q.table, 0xFF, 8 * L.cap, s);
        const int64_t n = na + nb;
        if (n) {
            join_hash_kernel<<<(unsigned)std::min<int64_t>(num_sms() * 16, blocks_for(n, 256 * ITEMS)), 256, 0, s>>>(q);
            count_launch();
        }
        trace_mark(s, "join:hash");
        // the number of distinct signatures bounds the sort's key bits
        unsigned long long hc0[4] = {0, 0, 0, 0};
        cudaMemcpyAsync(hc0, counters, sizeof(hc0), cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) return DW_E_CUDA;
        if (hc0[0]) return DW_E_WORKSPACE;  // more distinct signatures than the table holds
        const int64_t D = L.D;  // ids are table slots + 1
        const int nbits = bits_for(D);
        int32_t *first_a = (int32_t *)(base + L.first_a), *end_a = (int32_t *)(base + L.end_a);
        int32_t *first_b = (int32_t *)(base + L.first_b), *end_b = (int32_t *)(base + L.end_b);
        uint32_t *sid_a = (uint32_t *)(base + L.sid_a), *sid_b = (uint32_t *)(base + L.sid_b);
        uint32_t *six_a = (uint32_t *)(base + L.six_a), *six_b = (uint32_t *)(base + L.six_b);
        cudaMemsetAsync(end_a, 0, 4 * D, s);
        cudaMemsetAsync(end_b, 0, 4 * D, s);
        size_t cb = L.cub_bytes;
        if (na) {  // stable: equal ids keep op order
            cub::DeviceRadixSort::SortPairs(base + L.cub, cb, q.id_a, sid_a, q.ix_a, six_a, (int)na, 0, nbits, s);
            trace_mark(s, "join:sort_a");
            run_bounds_kernel<<<blocks_for(na, 256 * RB_ITEMS), 256, 0, s>>>(sid_a, na, first_a, end_a);
            count_launch(4);
            trace_mark(s, "join:bounds_a");
        }
        if (nb) {
            cb = L.cub_bytes;
            cub::DeviceRadixSort::SortPairs(base + L.cub, cb, q.id_b, sid_b, q.ix_b, six_b, (int)nb, 0, nbits, s);
            trace_mark(s, "join:sort_b");
            run_bounds_kernel<<<blocks_for(nb, 256 * RB_ITEMS), 256, 0, s>>>(sid_b, nb, first_b, end_b);
            count_launch(4);
            trace_mark(s, "join:bounds_b");
        }
        if (na) {
            unsigned int *cursor = (unsigned int *)(base + L.pair_cursor);
            uint2 *stage = (uint2 *)(base + L.pair_stage);
            cudaMemsetAsync(cursor, 0, 4 * PAIR_MAXB, s);
            join_pair_bucket_kernel<<<blocks_for(na, PAIR_THREADS * PAIR_ITEMS), PAIR_THREADS, 0, s>>>(
                sid_a, six_a, na, first_a, six_b, first_b, end_b, cursor, stage);
            trace_mark(s, "join:pair_bucket");
            unsigned int *cursor2 = (unsigned int *)(base + L.win_cursor);
            uint2 *stage2 = (uint2 *)(base + L.win_stage);
            const int64_t nwin = (na + WIN_OPS - 1) / WIN_OPS;
            cudaMemsetAsync(cursor2, 0, 4 * nwin, s);
            join_pair_sub_kernel<<<(unsigned)((na + SUB_CHUNK - 1) / SUB_CHUNK), 256, 0, s>>>(stage, na, cursor2, stage2);
            count_launch(1);
            trace_mark(s, "join:pair_sub");
        }
        int32_t *bonly_tmp = (int32_t *)(base + L.bonly_tmp);
        if (nb) {
            join_bonly_kernel<<<blocks_for(D), 256, 0, s>>>(D, six_b, first_b, end_b, first_a, end_a, bonly_tmp, n_bonly);
            count_launch();
            trace_mark(s, "join:bonly");
        }
        unsigned long long hc[4] = {0, 0, 0, 0};  // overflow, matched, next_id, n_bonly
        cudaMemcpyAsync(hc, counters, sizeof(hc), cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) return DW_E_CUDA;
        b_only = (int64_t)(unsigned int)hc[3];
        if (b_only) {  // B-only operators in B order
            cb = L.cub_bytes;
            cub::DeviceRadixSort::SortKeys(base + L.cub, cb, bonly_tmp, d_b_only, (int)b_only, 0,
                                           bits_for(nb), s);
            count_launch(4);
            trace_mark(s, "join:bonly_sort");
        }

        if (n_bonly_io) *n_bonly_io = b_only;
    } else {
        b_only = n_bonly_io ? *n_bonly_io : 0;
    }
    if (!(phase & 2)) {
        DW_CHECK_LAUNCH();
        return DW_OK;
    }
    JoinSideDev A{a->d_start, a->d_end, a->d_rank, a->d_joules, a->d_work};
    JoinSideDev B{b->d_start, b->d_end, b->d_rank, b->d_joules, b->d_work};
    FindCols o = cols_of(out);
    // the matched count is this phase's own: a JoinPrep may be reused (other
    // threshold or ledgers), so it restarts from zero on every call
    cudaMemsetAsync(counters + 1, 0, sizeof(unsigned long long), s);
    if (na) {
        const uint2 *stage2 = (const uint2 *)(base + L.win_stage);
        const int64_t nwin = (na + WIN_OPS - 1) / WIN_OPS;
        const size_t smem = 4 * (size_t)WIN_OPS;
        cudaFuncSetAttribute(join_window_findings_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(join_window_findings_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        join_window_findings_kernel<<<(unsigned)nwin, WF_THREADS, smem, s>>>(stage2, na, d_match_a, A, B, threshold,
                                                                            o, d_epw_a, d_epw_b, counters + 1);
        count_launch();
        trace_mark(s, "join:findings_a");
    }
    if (b_only) {
        join_findings_b_kernel<<<blocks_for(b_only), 256, 0, s>>>(na, b_only, d_b_only, B, threshold, o,
                                                                   d_epw_a, d_epw_b);
        count_launch();
    }
    // {P, matched, A-only, B-only} written on the device: no host round trip
    join_count_kernel<<<1, 32, 0, s>>>(counters + 1, na, b_only, d_count);
    count_launch();
    trace_mark(s, "join:end");
    DW_CHECK_LAUNCH();
    return DW_OK;
}

int dw_join_diff(const dw_join_side_t *a, const dw_join_side_t *b, int64_t max_distinct, double threshold,
                 dw_findings_t *out, int32_t *d_match_a, int32_t *d_b_only, double *d_epw_a,
                 double *d_epw_b, int64_t *d_count, void *d_workspace, size_t workspace_bytes,
                 dw_stream_t stream) {
    int64_t nb_only = 0;
    return join_impl(a, b, max_distinct, threshold, out, d_match_a, d_b_only, d_epw_a, d_epw_b, d_count,
                     d_workspace, workspace_bytes, stream, 3, &nb_only);
}

int dw_join_prepare(const dw_join_side_t *a, const dw_join_side_t *b, int64_t max_distinct, int32_t *d_match_a,
                    int32_t *d_b_only, int64_t *n_b_only, void *d_workspace, size_t workspace_bytes,
                    dw_stream_t stream) {
    if (!n_b_only) return DW_E_ARG;
    return join_impl(a, b, max_distinct, 0.1, nullptr, d_match_a, d_b_only, nullptr, nullptr, nullptr, d_workspace,
                     workspace_bytes, stream, 1, n_b_only);
}

int dw_join_findings(const dw_join_side_t *a, const dw_join_side_t *b, int64_t max_distinct, double threshold,
                     dw_findings_t *out, int32_t *d_match_a, int32_t *d_b_only, int64_t n_b_only, double *d_epw_a,
                     double *d_epw_b, int64_t *d_count, void *d_workspace, size_t workspace_bytes,
                     dw_stream_t stream) {
    return join_impl(a, b, max_distinct, threshold, out, d_match_a, d_b_only, d_epw_a, d_epw_b, d_count, d_workspace,
                     workspace_bytes, stream, 2, &n_b_only);
}


size_t dw_rank_segmented_workspace_size(int32_t nseg, int64_t k) {
    if (nseg < 0) return 0;
    const int64_t cap = SEG_SORT_MAX;
    (void)k;
    size_t off = 0;
    off += au(sizeof(SegDesc) * (size_t)std::max(nseg, 1));
    off += au(sizeof(SegState) * (size_t)std::max(nseg, 1));
    off += au(4 * (size_t)HIST_BINS * std::max(nseg, 1));
    off += au(64);                                     // pending, overflow
    off += au(4 * (size_t)std::max(nseg, 1));          // cand_n
    off += au(24 * (size_t)cap * std::max(nseg, 1));   // candidates
    off += au(24 * (size_t)1024 * std::max(nseg, 1));  // waste partials (<= 1024 blocks per segment)
    return off;
}

int dw_rank_segmented(const dw_rank_segment_t *segs, int32_t nseg, int64_t k, int64_t *d_order,
                      double *d_summary, void *d_workspace, size_t workspace_bytes, dw_stream_t stream) {
    if (nseg < 0 || k < 0 || k > SEG_SORT_MAX || (nseg && !segs) || !d_workspace) return DW_E_ARG;
    if (nseg == 0) return DW_OK;
    if (workspace_bytes < dw_rank_segmented_workspace_size(nseg, k)) return DW_E_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t cap = SEG_SORT_MAX;
    std::vector<SegDesc> h(nseg);
    int64_t pmax = 0;
    for (int i = 0; i < nseg; ++i) {
        const dw_rank_segment_t &g = segs[i];
        if (g.P < 0 || (g.P && !g.d_key_hi)) return DW_E_ARG;
        h[i] = SegDesc{g.d_key_hi, g.d_key_lo, g.d_tie_rank, g.n_a, g.P, std::min(k, g.P)};
        pmax = std::max(pmax, g.P);
    }
    if (k && !d_order) return DW_E_ARG;
    char *base = (char *)d_workspace;
    size_t off = 0;
    SegDesc *d_segs = (SegDesc *)(base + off); off += au(sizeof(SegDesc) * nseg);
    SegState *st = (SegState *)(base + off); off += au(sizeof(SegState) * nseg);
    unsigned *hist = (unsigned *)(base + off); off += au(4 * (size_t)HIST_BINS * nseg);
    unsigned *flags = (unsigned *)(base + off); off += au(64);
    unsigned *cand_n = (unsigned *)(base + off); off += au(4 * (size_t)nseg);
    uint64_t *chi = (uint64_t *)(base + off);
    uint64_t *clo = chi + cap * nseg;
    int64_t *cidx = (int64_t *)(clo + cap * nseg);
    off += au(24 * (size_t)cap * nseg);
    unsigned long long *partials = (unsigned long long *)(base + off);
    cudaMemcpyAsync(d_segs, h.data(), sizeof(SegDesc) * nseg, cudaMemcpyHostToDevice, s);
    // blocks per segment: about num_sms * 8 blocks in all, <= 1024 per segment
    const int64_t want = std::max<int64_t>(1, (int64_t)num_sms() * 8 / nseg);
    const unsigned bps = (unsigned)std::max<int64_t>(1, std::min<int64_t>({want, 1024, blocks_for(pmax, SEG_BLOCK)}));
    seg_init_kernel<<<(nseg + 255) / 256, 256, 0, s>>>(d_segs, nseg, st, hist, cand_n, flags);
    cudaMemsetAsync(flags, 0, 64, s);
    count_launch();
    if (d_summary) {
        seg_waste_kernel<<<dim3(bps, nseg), 256, 0, s>>>(d_segs, partials);
        seg_waste_final_kernel<<<nseg, 32, 0, s>>>(d_segs, partials, (int)bps, d_summary);
        count_launch(2);
    }
    if (k == 0) {
        DW_CHECK_LAUNCH();
        return DW_OK;
    }
    for (int round = 0; round < 128 / HIST_BITS; ++round) {
        seg_hist_kernel<<<dim3(bps, nseg), SEG_BLOCK, 0, s>>>(d_segs, st, hist);
        seg_select_kernel<<<nseg, 32, 0, s>>>(d_segs, st, hist, cap, flags);
        count_launch(2);
        unsigned pending = 0;
        cudaMemcpyAsync(&pending, flags, 4, cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) return DW_E_CUDA;
        if (!pending) break;
        cudaMemsetAsync(flags, 0, 4, s);
    }
    seg_compact_kernel<<<dim3(bps, nseg), 256, 0, s>>>(d_segs, st, cap, chi, clo, cidx, cand_n);
    const size_t smem = 24 * (size_t)cap;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(seg_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    seg_sort_kernel<<<nseg, SEG_SORT_THREADS, smem, s>>>(d_segs, cap, chi, clo, cidx, cand_n, k, d_order,
                                                          (int *)(flags + 1));
    count_launch(2);
    int overflow = 0;
    cudaMemcpyAsync(&overflow, flags + 1, 4, cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return DW_E_CUDA;
    if (overflow) return DW_E_WORKSPACE;  // massive ties at a threshold key (cannot happen: keys are distinct)
    DW_CHECK_LAUNCH();
    return DW_OK;
}


int dw_topk_rows(const int64_t *d_order, int64_t k, int64_t n_a, const int32_t *d_match_a, const int32_t *d_b_only,
                 const double *d_joules_a, const double *d_joules_b, const int64_t *d_start_a,
                 const int64_t *d_end_a, const int64_t *d_start_b, const int64_t *d_end_b, int64_t *d_out,
                 dw_stream_t stream) {
    if (k < 0 || n_a < 0 || (k && (!d_order || !d_out))) return DW_E_ARG;
    if (k) {
        topk_rows_kernel<<<(unsigned)ceil_div(k, 128), 128, 0, (cudaStream_t)stream>>>(
            d_order, k, n_a, d_match_a, d_b_only, d_joules_a, d_joules_b, d_start_a, d_end_a, d_start_b, d_end_b,
            d_out);
        count_launch();
    }
    DW_CHECK_LAUNCH();
    return DW_OK;
}

}  // extern "C"
