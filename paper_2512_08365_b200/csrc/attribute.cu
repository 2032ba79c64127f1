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
#include <cstring>
#include <algorithm>
#include <type_traits>

#include <cub/cub.cuh>

#include "dw_common.cuh"

namespace dw {

constexpr int TILE = DW_TILE;                // segments per tile
constexpr int DIRECT = DW_DIRECT_MAX;        // sequential-sum cap
constexpr int WIN = TILE + DIRECT + 6;       // window slots: 2 halo + TILE + DIRECT + 2, + virtual end
constexpr int ATTR_THREADS = DW_TILE_THREADS; // threads of one consumer group
constexpr int ATTR_WARPS = ATTR_THREADS / 32;
#ifndef DW_GROUPS
#define DW_GROUPS 4
#endif
constexpr int GROUPS = DW_GROUPS;            // consumer groups per CTA (tiles processed concurrently)
#ifndef DW_STAGES
#define DW_STAGES 5
#endif
constexpr int STAGES = DW_STAGES;            // TMA ring depth (tiles staged per CTA)
constexpr int CTAS_PER_SM = 1;

#ifdef DW_PHASE_PROF
// diagnostic build only: cycles per tile phase, summed over consumer groups
// (thread 0 of each group) and the producer; read with dw_phase_prof()
__device__ unsigned long long g_phase[16];
#define PROF(i)                                                                 \
    do {                                                                        \
        if (ctid == 0) {                                                        \
            long long t_ = clock64();                                           \
            atomicAdd(&g_phase[i], (unsigned long long)(t_ - prof_t));          \
            prof_t = t_;                                                        \
        }                                                                       \
    } while (0)
#else
#define PROF(i) do { (void)prof_t; } while (0)
#endif

struct AttrParams {
    const int64_t *ts;
    const double *w;
    int64_t S;
    int64_t span_hi;  // step: end of the last segment
    int64_t ntiles;
    int32_t kind;
    int32_t nsets;
    int32_t validate_order;
    int32_t sum_mode;            // DW_SUM_REFERENCE | DW_SUM_EXACT
    const int64_t *start[DW_MAX_SETS];
    const int64_t *end[DW_MAX_SETS];
    double *out[DW_MAX_SETS];
    const int64_t *perm[DW_MAX_SETS];  // sorted position -> caller index (unsorted sets)
    int64_t n[DW_MAX_SETS];
    int32_t check_sorted[DW_MAX_SETS];
    const int64_t *first;        // [nsets][ntiles + 1]
    unsigned long long *tile_fx; // [ntiles][2] exact int128 tile sums: sum of q(piece) over the tile
    unsigned long long *prefix;  // [ntiles + 1][2] exact int128 prefix of the tile sums
    unsigned long long *scan_part; // [nblocks][2] scan partials
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
    return __dadd_rn(wa, __dsub_rn(w(j), wa));  // frac == 1.0 exactly
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
    if (t < 4) {
        st->totals[t] = 0.0;
        st->pad[t] = 0;  // every byte of the block defined (dw_status copies all of it)
    }
}

// ------------------------------------------------------------ K1 partition
// Every PIDX_STRIDE-th interval start of each set: a ~1 MB index the
// partition searches first (L2-resident), so each tile boundary costs a
// handful of DRAM sectors instead of a full-depth search over the starts.
#ifndef DW_PIDX_STRIDE
#define DW_PIDX_STRIDE 1024
#endif
constexpr int64_t PIDX_STRIDE = DW_PIDX_STRIDE;

struct PartIndex {
    int64_t *p[DW_MAX_SETS];
};

__global__ void partition_index_kernel(AttrParams p, PartIndex idx, int nsets) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (int j = 0; j < nsets; ++j) {
        const int64_t m = ceil_div(p.n[j], PIDX_STRIDE);
        if (i < m) idx.p[j][i] = __ldg(p.start[j] + i * PIDX_STRIDE);
    }
}

__global__ void partition_kernel(AttrParams p, PartIndex idx) {
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
        // first k with a[k] >= key: bisect the sampled index (cached), then
        // the PIDX_STRIDE-wide bracket of the starts it leaves
        const int64_t key = p.ts[b * TILE];
        const int64_t *a = p.start[j];
        const int64_t *ix = idx.p[j];
        int64_t lo = 0, hi = ceil_div(n, PIDX_STRIDE);  // first index entry >= key
        while (lo < hi) {
            const int64_t mid = lo + ((hi - lo) >> 1);
            if (__ldg(ix + mid) < key) lo = mid + 1; else hi = mid;
        }
        // a[(lo-1)*STRIDE] < key (lo > 0), a[lo*STRIDE] >= key (if in range)
        int64_t l2 = lo > 0 ? (lo - 1) * PIDX_STRIDE + 1 : 0;
        int64_t h2 = lo * PIDX_STRIDE < n ? lo * PIDX_STRIDE : n;
        while (l2 < h2) {
            const int64_t mid = l2 + ((h2 - l2) >> 1);
            if (__ldg(a + mid) < key) l2 = mid + 1; else h2 = mid;
        }
        r = l2;
    }
    const_cast<int64_t *>(p.first)[j * nb + b] = r;
}

// --------------------------------------------------------- K2 tile kernel
// Warp-specialised persistent kernel.  Warp NCW (the producer) walks this
// CTA's tiles STAGES ahead of the consumers: it reads the tile's interval
// ranges from the partition, and with 1-D TMA (cp.async.bulk, completion on
// the stage's `full` mbarrier) stages (a) the sample window and (b) every
// set's [start, end) columns of the intervals that begin in the tile.  The
// NCW consumer warps wait on `full`, integrate, and release the stage through
// `empty`.  No consumer ever waits on a global load in the common case.
constexpr int NCW = ATTR_WARPS;              // warps per consumer group
#ifndef DW_NPROD
#define DW_NPROD 1
#endif
constexpr int NPROD = DW_NPROD;              // producer warps
constexpr int KTHREADS = GROUPS * ATTR_THREADS + 32 * NPROD;
#ifndef DW_IV_POOL
#define DW_IV_POOL 384
#endif
constexpr int IV_POOL = DW_IV_POOL;          // staged intervals per stage (all sets)

struct StageMeta {
    int64_t wb;                 // window base (global sample index)
    int64_t f0[DW_MAX_SETS];    // first interval of the tile, per set
    int64_t c[DW_MAX_SETS + 1]; // cumulative interval counts over sets
    int64_t a0[DW_MAX_SETS];    // staged copy starts at this (even) interval index
    int32_t copied[DW_MAX_SETS];
    int32_t pool[DW_MAX_SETS];
    int32_t cnt;                // samples in the window
};

template <int NST, int NWIN>
struct __align__(16) TileSmemT {  // the stage ring, shared by the producer and every group
    static constexpr int kStages = NST;
    static constexpr int kWin = NWIN;
    int64_t ts[NST][NWIN];
    double w[NST][NWIN];
    int64_t iv_lo[NST][IV_POOL];
    int64_t iv_hi[NST][IV_POOL];
    StageMeta meta[NST];
    uint64_t full[NST];
    uint64_t empty[NST];
    int claim;                  // next position of this CTA's tile sequence to hand to a group
};
using TileSmem = TileSmemT<STAGES, WIN>;

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// named barrier over one consumer group (the producer never joins)
__device__ __forceinline__ void consumer_sync(int g) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(ATTR_THREADS) : "memory");
}

template <int HALO = DIRECT>
__device__ __forceinline__ void tile_window(int64_t tile, int64_t S, int64_t &wb, int64_t &we) {
    wb = tile * TILE - 2;
    if (wb < 0) wb = 0;
    we = (tile + 1) * TILE + HALO + 2;  // keeps the steady-state window even (16-B TMA)
    if (we > S) we = S;
}

// joules = tot / 1e6, correctly rounded: Markstein's final step with the
// correctly rounded reciprocal (one multiply + two FMAs instead of a full
// software division; bit-identical to IEEE division for these operands).
__device__ __forceinline__ double div_1e6(double x) {
    const double inv = 1.0 / US_PER_S;
    double q = __dmul_rn(x, inv);
    double r = __fma_rn(-q, US_PER_S, x);
    return __fma_rn(r, inv, q);
}

__device__ __forceinline__ void report_bad(const AttrParams &p, int j, int64_t k) {
    int64_t idx = p.perm[j] ? __ldg(p.perm[j] + k) : k;
    atomic_min_index(&p.st->bad_index[j], idx);
}

__device__ __forceinline__ void push_long(const AttrParams &p, int j, int64_t k) {
    unsigned long long slot = atomicAdd(&p.st->long_count, 1ULL);
    p.long_list[slot] = ((unsigned long long)j << 56) | (unsigned long long)k;
}

// Timestamps of the current window, relative to its first sample: uint32 for
// narrow windows (span < 2^32 us, the common case: 32-bit loads and math),
// int64 otherwise.  Index r is window-relative (global index = wb + r); slot
// cnt holds the virtual end of the last step segment when the window reaches S.
struct Ts32 {
    const uint32_t *t;
    __device__ __forceinline__ uint32_t operator()(int r) const { return t[r]; }
};
struct Ts64 {
    const int64_t *t;
    int64_t base;
    __device__ __forceinline__ int64_t operator()(int r) const { return t[r] - base; }
};

// last r in [r0, r1) with ts(r) <= key, given ts(r0) <= key.  Starts at an
// interpolated guess (uniform grids hit in 1-2 probes) and gallops.
template <typename TS, typename T>
__device__ __forceinline__ int search_last_le(const TS &ts, int r0, int r1, T key, float scale) {
    int g = r0 + (int)((float)(key - ts(r0)) * scale);
    g = g < r0 ? r0 : (g >= r1 ? r1 - 1 : g);
    int lo, hi;  // invariant: ts(lo) <= key, ts(hi) > key or hi == r1
    if (ts(g) <= key) {
        lo = g;
        int step = 1;
        hi = lo + 1;
        while (hi < r1 && ts(hi) <= key) {
            lo = hi;
            step <<= 1;
            hi = lo + step;
        }
        if (hi > r1) hi = r1;
    } else {
        hi = g;
        int step = 1;
        lo = hi - 1;
        while (lo > r0 && ts(lo) > key) {
            hi = lo;
            step <<= 1;
            lo = hi - step;
        }
        if (lo < r0) lo = r0;
    }
    while (hi - lo > 1) {
        int m = (lo + hi) >> 1;
        if (ts(m) <= key) lo = m; else hi = m;
    }
    return lo;
}

// One interval of a STEP signal over the staged window: the reference's
// sequential sum (energy.py:99-104) with the zero-overlap segments skipped
// (they add nothing there either).  Returns false when it spans > DIRECT
// segments (the fixed-point path takes it).
template <typename TS, typename T>
__device__ __forceinline__ bool step_interval(const TS &ts, const double *w, int r0, int r1,
                                              T lo, T hi, float scale, double &tot) {
    if (hi == lo) { tot = 0.0; return true; }
    int i = search_last_le(ts, r0, r1, lo, scale);
    T e = ts(i + 1);
    if (hi <= e) {  // single segment
        tot = __dmul_rn(w[i], (double)(hi - lo));
        return true;
    }
    tot = __dmul_rn(w[i], (double)(e - lo));
    int nseg = 1;
    ++i;
    T s = e;
    e = ts(i + 1);
    while (e < hi) {
        if (nseg == DIRECT) return false;
        tot = __dadd_rn(tot, __dmul_rn(w[i], (double)(e - s)));
        ++nseg;
        ++i;
        s = e;
        e = ts(i + 1);
    }
    if (nseg == DIRECT) return false;
    tot = __dadd_rn(tot, __dmul_rn(w[i], (double)(hi - s)));
    return true;
}

// v(t) of energy.py:115-124 for an interior sample j (1 <= j <= S-2): the
// first bracketing pair is (j-1, j) with frac == 1.0 exactly, so
// ws[j-1] + 1.0*(ws[j]-ws[j-1]) == ws[j-1] + (ws[j]-ws[j-1]).
__device__ __forceinline__ double lin_interior(const double *w, int r) {
    double wa = w[r - 1];
    return __dadd_rn(wa, __dsub_rn(w[r], wa));
}

// One interval of a LINEAR (sampled) signal: trapezoid over
// [lo] + {ts in (lo, hi)} + [hi] (energy.py:126-130).
template <typename TS, typename T>
__device__ __forceinline__ bool linear_interval(const TS &ts, const double *w, int r0, int r1,
                                                int rcnt, T lo, T hi, int64_t glo, int64_t ghi,
                                                int64_t ts0, int64_t tsl, double w0, double wl,
                                                float scale, double &tot) {
    int a = search_last_le(ts, r0, r1, lo, scale);
    int first = a + 1;  // first window index with ts > lo
    double vprev;
    if (glo <= ts0) {
        vprev = w0;
    } else if (glo >= tsl) {
        vprev = wl;
    } else {
        int i = (ts(a) == lo) ? a - 1 : a;  // first bracketing pair (i, i+1)
        double wa = w[i];
        double frac = __ddiv_rn((double)(lo - ts(i)), (double)(ts(i + 1) - ts(i)));
        vprev = __dadd_rn(wa, __dmul_rn(frac, __dsub_rn(w[i + 1], wa)));
    }
    T prev = lo;
    tot = 0.0;
    int j = first;
    int m = 0;
    while (j < rcnt && ts(j) < hi) {
        if (m == DIRECT - 1) return false;  // pieces = interior + 1 > DIRECT
        double vj = lin_interior(w, j);
        T tj = ts(j);
        tot = __dadd_rn(tot, __dmul_rn(__dmul_rn(0.5, __dadd_rn(vprev, vj)), (double)(tj - prev)));
        prev = tj;
        vprev = vj;
        ++j;
        ++m;
    }
    double vh;
    if (ghi <= ts0) {
        vh = w0;
    } else if (ghi >= tsl) {
        vh = wl;
    } else {
        int i = j - 1;  // ts(j-1) < hi <= ts(j)
        double wa = w[i];
        double frac = __ddiv_rn((double)(hi - ts(i)), (double)(ts(i + 1) - ts(i)));
        vh = __dadd_rn(wa, __dmul_rn(frac, __dsub_rn(w[i + 1], wa)));
    }
    tot = __dadd_rn(tot, __dmul_rn(__dmul_rn(0.5, __dadd_rn(vprev, vh)), (double)(hi - prev)));
    return true;
}

struct TileCtx {
    int64_t ts0, tsl, span_lo, span_hi, base;
    double w0, wl;
    float scale;
};

template <int KIND, typename TS, typename T>
__device__ __forceinline__ void tile_intervals(const AttrParams &p, const TileSmem &sm, int stage,
                                               const TS &ts, const double *w, int64_t tile,
                                               T sat, const TileCtx &cx, int ctid) {
    const StageMeta &M = sm.meta[stage];
    const int64_t S = p.S;
    const int64_t wb = M.wb;
    const int r0 = (int)(tile * TILE - wb);
    const int r1 = (int)(min((tile + 1) * TILE, S) - wb);
    const int rcnt = M.cnt;
    const int64_t total = M.c[DW_MAX_SETS];
    for (int64_t v = ctid; v < total; v += ATTR_THREADS) {
        const int j = (v >= M.c[1]) + (v >= M.c[2]) + (v >= M.c[3]);
        const int64_t k = v - M.c[j] + M.f0[j];
        const int64_t idx = k - M.a0[j];
        int64_t glo, ghi;
        if (idx < M.copied[j]) {
            glo = sm.iv_lo[stage][M.pool[j] + idx];
            ghi = sm.iv_hi[stage][M.pool[j] + idx];
        } else {
            glo = __ldg(p.start[j] + k);
            ghi = __ldg(p.end[j] + k);
        }
        if (p.check_sorted[j] && k > 0) {
            const int64_t pidx = idx - 1;
            const int64_t prev = (pidx >= 0 && pidx < M.copied[j])
                                     ? sm.iv_lo[stage][M.pool[j] + pidx]
                                     : __ldg(p.start[j] + k - 1);
            if (prev > glo) atomic_min_index(&p.st->unsorted_index[j], k);
        }
        if (ghi < glo || glo < cx.span_lo || ghi > cx.span_hi) {
            report_bad(p, j, k);
            continue;
        }
        // window-relative times; hi beyond the window saturates (the interval
        // is then long and leaves through the DIRECT cap)
        const T lo = (T)(glo - cx.base);
        const int64_t dh = ghi - cx.base;
        const T hi = dh > (int64_t)sat ? sat : (T)dh;
        double tot;
        bool ok;
        if (KIND == DW_SIGNAL_STEP)
            ok = step_interval(ts, w, r0, r1, lo, hi, cx.scale, tot);
        else
            ok = linear_interval(ts, w, r0, r1, rcnt, lo, hi, glo, ghi, cx.ts0, cx.tsl, cx.w0,
                                 cx.wl, cx.scale, tot);
        if (!ok) {
            push_long(p, j, k);
        } else {
            const int64_t oidx = p.perm[j] ? __ldg(p.perm[j] + k) : k;
            p.out[j][oidx] = div_1e6(tot);
        }
    }
}

// ---- narrow tiles: precomputed terms, two phases ----
// Pass A writes the window's 32-bit relative timestamps (group smem) and then
// every interior integrand term of the tile's pieces into the stage's int64
// timestamp slots (no longer needed once ts32 exists); the tile sum is folded
// from those same terms.  Phase 1 (concurrent with the terms: it only needs
// ts32) finds, per interval, its first piece a and its interior-term count,
// and evaluates the two edge pieces (the only ones that depend on lo / hi:
// the interpolated endpoint values and their divisions).  Phase 2 folds
// F0 + term[a+1] + ... + L in the reference's order: one shared load and one
// dependent add per step.  (A counting sort by length to cut lane divergence
// in phase 2 was measured and dropped: on C4 its histogram, scan, scatter and
// two extra barriers cost more than the divergence it removes.)
#ifndef DW_CHUNK
#define DW_CHUNK 512
#endif
constexpr int CHUNK = DW_CHUNK;  // intervals per phase-1/phase-2 round
#ifndef DW_FOLD_UNROLL
#define DW_FOLD_UNROLL 4
#endif
constexpr int FOLD_UNROLL = DW_FOLD_UNROLL;

// item meta: q (chunk index, 10 bits) | s (first interior term, 11 bits) << 10 |
//            cnt (interior terms, 9 bits) << 21 | has_last << 30
static_assert(CHUNK <= 1024 && WIN <= 2048 && DIRECT < 512, "item meta packing");

struct __align__(16) GroupSmem {  // private to one consumer group
    uint32_t ts32[WIN];
    double F0[CHUNK];    // first piece (0.0 + first piece for the trapezoid)
    double L[CHUNK];     // last piece
    uint32_t meta[CHUNK];
    unsigned long long red[NCW][2];
    int64_t kq[2][DW_MAX_SETS];  // per chunk parity, per set: interval index = kq + chunk index
    int4 desc[2][DW_MAX_SETS];   // per chunk parity, per set: smem base, staged limit, first staged slot
    int next_it;              // the group's claimed next tile (sequence position)
};

// num / den correctly rounded, for integers 0 <= num <= den < 2^32 (the
// trapezoid's frac, energy.py:121).  Markstein's final step on a reciprocal
// refined to ~1 ulp: the pre-rounding error is < 2^-50 ulp, while a quotient
// of such integers is either exact or >= ulp / (4 den) > 2^-34 ulp away from
// a rounding midpoint, so the result equals IEEE division (scripts/micro/
// div_check.cu checks it against __ddiv_rn: exhaustive for den <= 4096 plus
// 4e9 random pairs).  About a third of __ddiv_rn's instructions, no branch.
__device__ __forceinline__ double div_u32(uint32_t num, uint32_t den) {
#ifdef DW_EXP_NODIV
    return (double)num * 0.01;
#endif
    const double b = (double)den, a = (double)num;
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(b));
    double e = __fma_rn(-b, y, 1.0);
    y = __fma_rn(y, e, y);
    e = __fma_rn(-b, y, 1.0);
    y = __fma_rn(y, e, y);
    const double q = __dmul_rn(a, y);
    const double r = __fma_rn(-q, b, a);
    return __fma_rn(r, y, q);
}

// item meta: q (chunk index, 9 bits) | s (first interior term, 11 bits) << 9 |
//            cnt (interior terms, 9 bits) << 20 | has_last << 29 | set << 30
__device__ __forceinline__ uint32_t pack_meta(int q, int s, int cnt, int last, int j) {
    return (uint32_t)q | ((uint32_t)s << 9) | ((uint32_t)cnt << 20) | ((uint32_t)last << 29) |
           ((uint32_t)j << 30);
}
constexpr uint32_t META_NONE = 0xFFFFFFFFu;  // no valid item packs to it (s < WIN < 2047, cnt <= DIRECT < 511)
static_assert(CHUNK <= 512, "meta q field is 9 bits");
static_assert(GROUPS < STAGES, "claims in flight must span fewer positions than the ring");

// last r in [r0, r1) with ts[r] <= key, given ts[r0] <= key and kref <= key
// (kref = ts[gref] or a time known to lie at or after it).  Probes the
// interpolated guess and its successor (independent loads); a miss (sample
// spacing not uniform) gallops from the guess, then bisects.
__device__ __forceinline__ int find_le(const uint32_t *ts, int r0, int r1, uint32_t key, uint32_t kref,
                                       int gref, float scale) {
    const float off = (float)(key - kref) * scale;
    int g = off >= (float)(r1 - 1 - gref) ? r1 - 1 : gref + (int)off;
    if (g < r0) g = r0;
    const uint32_t tg = ts[g], tn = ts[g + 1];
    if (tg <= key && (g + 1 >= r1 || tn > key)) return g;
    int lo, hi;  // ts[lo] <= key; ts[hi] > key or hi == r1
    if (tg <= key) {
        lo = g + 1;  // ts[g + 1] <= key here
        int step = 1;
        hi = lo + 1;
        while (hi < r1 && ts[hi] <= key) {
            lo = hi;
            step <<= 1;
            hi = lo + step;
        }
        if (hi > r1) hi = r1;
    } else {
        hi = g;
        int step = 1;
        lo = hi - 1;
        while (lo > r0 && ts[lo] > key) {
            hi = lo;
            step <<= 1;
            lo = hi - step;
        }
        if (lo < r0) lo = r0;
    }
    while (hi - lo > 1) {
        const int m = (lo + hi) >> 1;
        if (ts[m] <= key) lo = m; else hi = m;
    }
    return lo;
}

// find_le with a wider first probe: the four timestamps around the
// interpolated guess (independent loads), which settle a guess off by one
// either way -- a jittered clock's usual miss -- without the gallop.
__device__ __forceinline__ int find_le4(const uint32_t *ts, int r0, int r1, uint32_t key, uint32_t kref,
                                        int gref, float scale) {
    if (r1 - r0 >= 4) {
        const float off = (float)(key - kref) * scale;
        int g = off >= (float)(r1 - 2 - gref) ? r1 - 2 : gref + (int)off;
        g = g < r0 + 1 ? r0 + 1 : g;  // g - 1 >= r0, g + 1 <= r1 - 1
        const uint32_t tm = ts[g - 1], t0 = ts[g], t1 = ts[g + 1], t2 = ts[g + 2 < r1 ? g + 2 : g + 1];
        if (tm <= key && (g + 2 >= r1 || t2 > key)) return g - 1 + (t0 <= key) + (t1 <= key);
    }
    return find_le(ts, r0, r1, key, kref, gref, scale);
}

// Phase 1 for one interval (window-relative lo <= hi, lo in the tile): edge
// pieces and interior count.  Returns false when it spans more than DIRECT
// pieces (the fixed-point path takes it).  Branch-free apart from the
// search fallbacks.
template <int KIND, int CAP = DIRECT>
__device__ __forceinline__ bool phase1_item(const uint32_t *ts, const double *w, int r0, int r1, int cnt_win,
                                            uint32_t lo, uint32_t hi, bool lo_first, bool lo_last,
                                            bool hi_first, bool hi_last, const TileCtx &cx, double &F0,
                                            double &L, int &s, int &cnt, int &last) {
    const int a = find_le(ts, r0, r1, lo, ts[r0], r0, cx.scale);
    const int lim = min(a + CAP + 1, cnt_win);
    const uint32_t ta = ts[a], ta1 = ts[a + 1];
    s = a + 1;
    if (KIND == DW_SIGNAL_STEP) {
        // energy.py:99-104, zero-overlap segments skipped; b = last segment start < hi
        const int b = hi > lo ? find_le(ts, a, lim, hi - 1, ts[a], a, cx.scale) : a;
        const int n = hi > lo ? b - a + 1 : 0;  // segments
        if (n > CAP) return false;
        const double wa = w[a];
        F0 = n == 0 ? 0.0 : __dmul_rn(wa, (double)((n == 1 ? hi : ta1) - lo));
        L = __dmul_rn(w[b], (double)(hi - ts[b]));
        cnt = n >= 2 ? n - 2 : 0;
        last = n >= 2;
        return true;
    } else {
        // energy.py:108-130: points [lo] + {ts in (lo, hi)} + [hi]; b = last sample < hi
        const int b = ta < hi ? find_le(ts, a, lim, hi - 1, ta, a, cx.scale) : a - 1;
        const int m = b - a;  // -1 only when hi == lo == ts[a]
        if (m + 1 > CAP) return false;  // pieces = m + 1
        // v(lo), v(hi): first bracketing pair (energy.py:115-124)
        const int il = ta == lo && a > 0 ? a - 1 : a;  // (a == 0: lo is the first sample, vlo = w0)
        const double wl0 = w[il], wl1 = w[il + 1];
        const uint32_t tl0 = ts[il];
        const double vlo_i = __dadd_rn(wl0, __dmul_rn(div_u32(lo - tl0, ts[il + 1] - tl0), __dsub_rn(wl1, wl0)));
        const double vlo = lo_first ? cx.w0 : (lo_last ? cx.wl : vlo_i);
        const double wh0 = w[b], wh1 = w[b + 1];
        const uint32_t th0 = ts[b];
        const double vhi_i = __dadd_rn(wh0, __dmul_rn(div_u32(hi - th0, ts[b + 1] - th0), __dsub_rn(wh1, wh0)));
        const double vhi = hi_first ? cx.w0 : (hi_last ? cx.wl : vhi_i);
        // interior values v(a+1), v(b) (the loads are in range even when unused)
        const double wa0 = w[a], wa1 = w[a + 1];
        const double v1 = __dadd_rn(wa0, __dsub_rn(wa1, wa0));
        const double wbm = w[b > 0 ? b - 1 : 0];
        const double vb = __dadd_rn(wbm, __dsub_rn(wh0, wbm));
        const bool one = m <= 0;  // one piece [lo, hi]
        const double vn = one ? vhi : v1;
        const uint32_t tnx = one ? hi : ta1;
        F0 = __dadd_rn(0.0, __dmul_rn(__dmul_rn(0.5, __dadd_rn(vlo, vn)), (double)(tnx - lo)));
        L = __dmul_rn(__dmul_rn(0.5, __dadd_rn(vb, vhi)), (double)(hi - th0));
        cnt = one ? 0 : m - 1;
        last = !one;
        return true;
    }
}

// Per-set item descriptors of the chunk starting at c0 (one thread per set):
// item q of set j sits at smem index desc.x + q if q < desc.y (staged), and
// is interval kq + q of the set.
__device__ __forceinline__ void set_desc(const StageMeta &M, GroupSmem &so, int j, int64_t c0) {
    const int par = (int)((c0 / CHUNK) & 1);  // double-buffered: the previous chunk's phase 2 may still read
    const int64_t kq = M.f0[j] - M.c[j] + c0;            // interval index = kq + q
    const int64_t base = M.pool[j] + (kq - M.a0[j]);     // smem index = base + q
    const int64_t lim = M.a0[j] + M.copied[j] - kq;      // staged iff q < lim
    so.kq[par][j] = kq;
    auto clamp30 = [](int64_t v) -> int { return (int)(v < -(1LL << 30) ? -(1LL << 30) : (v > (1LL << 30) ? (1LL << 30) : v)); };
    so.desc[par][j] = make_int4(clamp30(base), clamp30(lim), M.pool[j], 0);
}

template <int KIND>
__device__ void tile_intervals_two_pass(const AttrParams &p, TileSmem &sm, GroupSmem &so, int stage,
                                      int64_t tile, const TileCtx &cx, int ctid, int g,
                                      long long &prof_t) {
    const StageMeta &M = sm.meta[stage];
    const int64_t S = p.S;
    const int64_t wb = M.wb;
    const int cnt_win = M.cnt;
    const int r0 = (int)(tile * TILE - wb);
    const int r1 = (int)(min((tile + 1) * TILE, S) - wb);
    const uint32_t *ts = so.ts32;
    const double *w = sm.w[stage];
    const double *term = reinterpret_cast<const double *>(sm.ts[stage]);
    const int64_t total = M.c[DW_MAX_SETS];
    const int nsets = p.nsets;
    (void)nsets;
    for (int64_t c0 = 0; c0 < total; c0 += CHUNK) {
        const int nch = (int)(total - c0 < CHUNK ? total - c0 : CHUNK);
        // ---- phase 1: locate, validate, edge pieces, bucket by length.  The
        // chunk's items (sets concatenated) are strided over the group's
        // threads, so every thread gets the same count whatever the set sizes.
        int cb1, cb2, cb3;  // chunk-relative set boundaries
        {
            auto rel = [&](int64_t c) -> int { return c <= c0 ? 0 : (c >= c0 + nch ? nch : (int)(c - c0)); };
            cb1 = rel(M.c[1]);
            cb2 = rel(M.c[2]);
            cb3 = rel(M.c[3]);
        }
        const int64_t *s_lo = sm.iv_lo[stage], *s_hi = sm.iv_hi[stage];
        const int par = (int)((c0 / CHUNK) & 1);
        const int4 *cdesc = so.desc[par];
        const int64_t *ckq = so.kq[par];
        for (int q = ctid; q < nch; q += ATTR_THREADS) {
            const int j = (q >= cb1) + (q >= cb2) + (q >= cb3);
            const int4 d = cdesc[j];  // {smem base, staged limit, smem first of the set}
            const int si = d.x + q;
            const bool staged = q < d.y;
            int64_t glo, ghi;
            if (staged) {
                glo = s_lo[si];
                ghi = s_hi[si];
            } else {
                const int64_t k = ckq[j] + q;
                glo = __ldg(p.start[j] + k);
                ghi = __ldg(p.end[j] + k);
            }
#ifndef DW_EXP_NOCHECK
            if (p.check_sorted[j]) {  // a set flagged sorted must be sorted by start
                int64_t prev;
                bool has_prev = true;
                if (staged && si > d.z) {
                    prev = s_lo[si - 1];
                } else {
                    const int64_t k = ckq[j] + q;
                    has_prev = k > 0;
                    prev = has_prev ? __ldg(p.start[j] + k - 1) : glo;
                }
                if (has_prev && prev > glo) atomic_min_index(&p.st->unsorted_index[j], ckq[j] + q);
            }
            if (ghi < glo || glo < cx.span_lo || ghi > cx.span_hi) {
                report_bad(p, j, ckq[j] + q);
                so.meta[q] = META_NONE;
                continue;
            }
#endif
            const uint32_t lo = (uint32_t)(glo - cx.base);
            const int64_t dh = ghi - cx.base;
            const uint32_t hi = dh > 0xFFFFFFFFLL ? 0xFFFFFFFFu : (uint32_t)dh;
            double F0, L;
            int s, cnt, last;
            if (!phase1_item<KIND>(ts, w, r0, r1, cnt_win, lo, hi, glo <= cx.ts0, glo >= cx.tsl,
                                   ghi <= cx.ts0, ghi >= cx.tsl, cx, F0, L, s, cnt, last)) {
                push_long(p, j, ckq[j] + q);
                so.meta[q] = META_NONE;
                continue;
            }
            so.F0[q] = F0;
            so.L[q] = L;
            so.meta[q] = pack_meta(q, s, cnt, last, j);

        }
        consumer_sync(g);
        PROF(3);
#ifdef DW_EXP_P1_ONLY
        consumer_sync(g);
        continue;
#endif
        // ---- phase 2: the interior folds, items in chunk order
        for (int q = ctid; q < nch; q += ATTR_THREADS) {
            const uint32_t mt = so.meta[q];
            if (mt == META_NONE) continue;
            const int s = (int)((mt >> 9) & 2047u);
            const int cnt = (int)((mt >> 20) & 511u);
            const int j = (int)(mt >> 30);
            double tot = so.F0[q];
            const double *tp = term + s;
#pragma unroll FOLD_UNROLL
            for (int u = 0; u < cnt; ++u) tot = __dadd_rn(tot, tp[u]);
            if ((mt >> 29) & 1u) tot = __dadd_rn(tot, so.L[q]);
            const int64_t k = ckq[j] + q;
            const int64_t oidx = p.perm[j] ? __ldg(p.perm[j] + k) : k;
            p.out[j][oidx] = div_1e6(tot);
        }
        if (ctid < DW_MAX_SETS && c0 + CHUNK < total) set_desc(M, so, ctid, c0 + CHUNK);
        consumer_sync(g);
        PROF(6);
    }
}

// Producer warp pw of NPROD handles positions it = pw, pw + NPROD, ... of
// this CTA's tile sequence (one tile per stage fill).  The partition bounds of
// 32 of its tiles are fetched at once (one global-load latency per 32 tiles)
// and handed out by shuffles; lane 0 waits for the slot, lays out the stage
// and arms the barrier, and the bulk copies are issued by separate lanes.
template <typename SM, int HALO = DIRECT>
__device__ __forceinline__ void producer(const AttrParams &p, SM &sm, int64_t span_hi, int pw) {
    constexpr int NST = SM::kStages;
    const int64_t S = p.S;
    const int lane = threadIdx.x & 31;
    const int64_t nb = p.ntiles + 1;
    const int ctid = lane;
    long long prof_t = clock64();
    for (int b0 = 0;; b0 += 32) {
        const int itb = pw + NPROD * b0;  // first position of this batch
        if ((int64_t)blockIdx.x + (int64_t)itb * gridDim.x >= p.ntiles) break;
        const int64_t tl = (int64_t)blockIdx.x + (int64_t)(itb + NPROD * lane) * gridDim.x;
        int64_t fl[DW_MAX_SETS], fh[DW_MAX_SETS];
#pragma unroll
        for (int j = 0; j < DW_MAX_SETS; ++j) {
            const bool ok = j < p.nsets && tl < p.ntiles;
            fl[j] = ok ? __ldg(p.first + j * nb + tl) : 0;
            fh[j] = ok ? __ldg(p.first + j * nb + tl + 1) : 0;
        }
        // lane u stages the u-th tile of the batch from its own registers
        for (int u = 0; u < 32; ++u) {
            const int it = itb + NPROD * u;
            const int64_t tile = (int64_t)blockIdx.x + (int64_t)it * gridDim.x;
            if (tile >= p.ntiles) break;
            if (lane == u) {
                const int stage = it % NST;
                StageMeta &M = sm.meta[stage];
                int64_t wb, we;
                tile_window<HALO>(tile, S, wb, we);
                const int cnt = (int)(we - wb);
                const int even = cnt & ~1;
                uint32_t bytes = 2u * 8u * (uint32_t)even;
                int64_t a0s[DW_MAX_SETS];
                int ms[DW_MAX_SETS], pools[DW_MAX_SETS];
                int pool = 0;
#pragma unroll
                for (int j = 0; j < DW_MAX_SETS; ++j) {
                    const int64_t f0 = fl[j], f1 = fh[j];
                    const int64_t a0 = f0 & ~(int64_t)1;
                    const int64_t want = f1 > f0 ? f1 - a0 : 0;
                    const int64_t room = IV_POOL - pool;
                    const int m = (int)(want < room ? want : room) & ~1;
                    a0s[j] = a0;
                    ms[j] = m;
                    pools[j] = pool;
                    pool += m;
                    bytes += 2u * 8u * (uint32_t)m;
                }
                PROF(8);
                if (it >= NST) mbar_wait(&sm.empty[stage], (uint32_t)(((it / NST) - 1) & 1));
                PROF(7);
                fence_proxy_async();
                M.wb = wb;
                M.cnt = cnt;
                M.c[0] = 0;
#pragma unroll
                for (int j = 0; j < DW_MAX_SETS; ++j) {
                    M.f0[j] = fl[j];
                    M.c[j + 1] = M.c[j] + (fh[j] - fl[j]);
                    M.a0[j] = a0s[j];
                    M.copied[j] = ms[j];
                    M.pool[j] = pools[j];
                }
                if (cnt & 1) {  // odd tail of the window: not a 16-byte multiple
                    sm.ts[stage][cnt - 1] = __ldg(p.ts + wb + cnt - 1);
                    sm.w[stage][cnt - 1] = __ldg(p.w + wb + cnt - 1);
                }
                if (wb + cnt == S) sm.ts[stage][cnt] = span_hi;  // virtual end of the last segment
                mbar_expect_tx(&sm.full[stage], bytes);
                if (even) {
                    tma_load_1d(sm.ts[stage], p.ts + wb, 8u * even, &sm.full[stage]);
                    tma_load_1d(sm.w[stage], p.w + wb, 8u * even, &sm.full[stage]);
                }
#pragma unroll
                for (int j = 0; j < DW_MAX_SETS; ++j) {
                    if (j < p.nsets && ms[j]) {
                        tma_load_1d(&sm.iv_lo[stage][pools[j]], p.start[j] + a0s[j], 8u * ms[j], &sm.full[stage]);
                        tma_load_1d(&sm.iv_hi[stage][pools[j]], p.end[j] + a0s[j], 8u * ms[j], &sm.full[stage]);
                    }
                }
            }
            __syncwarp();
        }
    }
}

// Terms of pieces r, r+1 for r = r0 + 2*ctid + 2*ATTR_THREADS*k, r < rend,
// stored to term[] (when non-null); returns this thread's exact share of the
// tile sum (q(piece) over its pieces < e1, int128; any grouping gives the
// same total).  Linear pieces use v(x) of energy.py:115-124 (w0 / wl at the
// signal's first / last sample, window indices rz0 / rzS; elsewhere the
// interior form w[x-1] + (w[x] - w[x-1])).
template <int KIND, typename WIDTH>
__device__ __forceinline__ i128 pair_terms(const double *w, const WIDTH &width, int r0, int rend, int e1,
                                           int rz0, int rzS, double w0, double wl, double *term, int ctid) {
    i128 acc = 0;
    for (int r = r0 + 2 * ctid; r < rend; r += 2 * ATTR_THREADS) {
        const double2 wr = *reinterpret_cast<const double2 *>(w + r);  // w[r], w[r+1]
        const double d0 = (double)width(r), d1 = (double)width(r + 1);
        double t0, t1;
        if (KIND == DW_SIGNAL_STEP) {
            t0 = __dmul_rn(wr.x, d0);
            t1 = __dmul_rn(wr.y, d1);
        } else {
            const double wm = w[r > 0 ? r - 1 : 0], w2 = w[r + 2];
            const double v0 = r == rz0 ? w0 : __dadd_rn(wm, __dsub_rn(wr.x, wm));
            const double v1 = __dadd_rn(wr.x, __dsub_rn(wr.y, wr.x));
            const double v1b = r + 1 == rzS ? wl : v1;
            const double v2 = r + 2 == rzS ? wl : __dadd_rn(wr.y, __dsub_rn(w2, wr.y));
            t0 = __dmul_rn(__dmul_rn(0.5, __dadd_rn(v0, v1b)), d0);
            t1 = __dmul_rn(__dmul_rn(0.5, __dadd_rn(v1, v2)), d1);
        }
        if (term) {
            if (r + 1 < rend) *reinterpret_cast<double2 *>(term + r) = make_double2(t0, t1);
            else term[r] = t0;
        }
        if (r < e1) acc += q40(t0);
        if (r + 1 < e1) acc += q40(t1);
    }
    return acc;
}

// exact int128 tile sum from each thread's share: warp sums to red[], then
// one thread adds the warps (after the group barrier that follows)
__device__ __forceinline__ void tile_fx_partial(i128 acc, unsigned long long (*red)[2], int ctid) {
    acc = warp_sum_i128(acc);
    if ((ctid & 31) == 0) {
        const I128Parts pp = split(acc);
        red[ctid >> 5][0] = pp.lo;
        red[ctid >> 5][1] = pp.hi;
    }
}
template <int NW>
__device__ __forceinline__ void tile_fx_store(const unsigned long long (*red)[2], unsigned long long *out) {
    i128 t = 0;
#pragma unroll
    for (int k = 0; k < NW; ++k) t += join(red[k][0], red[k][1]);
    const I128Parts pp = split(t);
    out[0] = pp.lo;
    out[1] = pp.hi;
}

struct Width32 {
    const uint32_t *t;
    __device__ __forceinline__ uint32_t operator()(int r) const { return t[r + 1] - t[r]; }
};
struct Width64 {
    const int64_t *t;
    __device__ __forceinline__ int64_t operator()(int r) const { return t[r + 1] - t[r]; }
};

template <int KIND>
__global__ void __launch_bounds__(KTHREADS, 1) attribute_tiles_kernel(AttrParams p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    TileSmem &sm = *reinterpret_cast<TileSmem *>(smem_raw);
    GroupSmem *groups =
        reinterpret_cast<GroupSmem *>(smem_raw + ((sizeof(TileSmem) + 15) & ~(size_t)15));
    const int tid = threadIdx.x;
    if ((int64_t)blockIdx.x >= p.ntiles) return;

    const int64_t S = p.S;
    TileCtx cx;
    cx.ts0 = __ldg(p.ts);
    cx.tsl = __ldg(p.ts + S - 1);
    cx.w0 = __ldg(p.w);
    cx.wl = __ldg(p.w + S - 1);
    cx.span_lo = cx.ts0;
    cx.span_hi = KIND == DW_SIGNAL_STEP ? p.span_hi : cx.tsl;
    const int64_t nterms = KIND == DW_SIGNAL_STEP ? S : S - 1;

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < GROUPS) groups[tid].next_it = tid;
    if (tid == 0) sm.claim = GROUPS;
    __syncthreads();

    if (tid >= GROUPS * ATTR_THREADS) {  // producer warps
        producer(p, sm, cx.span_hi, (tid - GROUPS * ATTR_THREADS) >> 5);
        return;
    }
    // Consumer groups claim positions of this CTA's tile sequence in order
    // (shared counter), so a group never waits on a stage two fills ahead of
    // an unconsumed one (claims in flight span < STAGES positions: GROUPS <
    // STAGES) and a slow tile does not hold up the others.
    const int g = tid / ATTR_THREADS;
    const int ctid = tid - g * ATTR_THREADS;
    GroupSmem &gs = groups[g];
    long long prof_t = clock64();
    for (;;) {
        const int it = gs.next_it;
        const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
        if (tile >= p.ntiles) break;
        const int stage = it % STAGES;
        mbar_wait(&sm.full[stage], (uint32_t)((it / STAGES) & 1));
        PROF(0);
#ifdef DW_SKIP_CONSUMERS
        consumer_sync(g);
        if (ctid == 0) {
            gs.next_it = atomicAdd(&sm.claim, 1);
            mbar_arrive(&sm.empty[stage]);
        }
        consumer_sync(g);
        continue;
#endif
        const StageMeta &M = sm.meta[stage];
        const int64_t wb = M.wb;
        const int cnt = M.cnt;
        const int64_t *s_ts = sm.ts[stage];
        const double *s_w = sm.w[stage];
        const int64_t base = s_ts[0];
        const int last = (wb + cnt == S) ? cnt : cnt - 1;
        const bool wide = (s_ts[last] - base) >= (int64_t)0xFFFFFFF0LL;
        const int r0 = (int)(tile * TILE - wb);
        const int r1 = (int)(min((tile + 1) * TILE, S) - wb);

        const int e1 = (int)(min((tile + 1) * TILE, nterms) - wb);
        const int rz0 = wb == 0 ? 0 : -1000;
        const int rzS = (S - 1 - wb) < (int64_t)WIN ? (int)(S - 1 - wb) : -1000;
        {
            const int64_t dt = s_ts[r1 < last ? r1 : last] - s_ts[r0];
            cx.scale = dt > 0 ? (float)(r1 - r0) / (float)dt : 0.0f;
        }
        cx.base = base;
        if (p.validate_order) {  // strictly increasing power timestamps (int64 compare)
            for (int r = r0 + ctid; r < r1 && wb + r + 1 < S; r += ATTR_THREADS)
                if (s_ts[r + 1] <= s_ts[r]) atomic_min_index(&p.st->order_index, wb + r);
        }
        if (ctid < DW_MAX_SETS) set_desc(M, gs, ctid, 0);  // published by the next barrier
        if (!wide) {
            // (a) 32-bit relative timestamps, two per thread
            for (int r = 2 * ctid; r <= last; r += 2 * ATTR_THREADS) {
                const longlong2 t2 = *reinterpret_cast<const longlong2 *>(s_ts + r);
                const uint32_t x = (uint32_t)(t2.x - base), y = (uint32_t)(t2.y - base);
                if (r + 1 <= last) *reinterpret_cast<uint2 *>(gs.ts32 + r) = make_uint2(x, y);
                else gs.ts32[r] = x;
            }
            consumer_sync(g);
            if (ctid == 0) gs.next_it = atomicAdd(&sm.claim, 1);  // every thread has read it
            PROF(1);
            // (b) interior terms of pieces r0 .. last-1 into the stage's ts slots
            // (phase 1 searches ts32 from here on), (c) the tile-sum partials
            double *term = reinterpret_cast<double *>(const_cast<int64_t *>(s_ts));
            const i128 acc = pair_terms<KIND>(s_w, Width32{gs.ts32}, r0, last, e1, rz0, rzS, cx.w0, cx.wl, term, ctid);
            tile_fx_partial(acc, gs.red, ctid);
            PROF(2);
            if (M.c[DW_MAX_SETS] == 0) consumer_sync(g);  // no intervals: red must still be visible
#ifdef DW_EXP_PASSA_ONLY
            consumer_sync(g);
#else
            tile_intervals_two_pass<KIND>(p, sm, gs, stage, tile, cx, ctid, g, prof_t);
#endif
            if (ctid == 0) tile_fx_store<NCW>(gs.red, p.tile_fx + 2 * tile);
        } else {
            const i128 acc = pair_terms<KIND>(s_w, Width64{s_ts}, r0, e1, e1, rz0, rzS, cx.w0, cx.wl,
                                              (double *)nullptr, ctid);
            tile_fx_partial(acc, gs.red, ctid);
            consumer_sync(g);
            if (ctid == 0) gs.next_it = atomicAdd(&sm.claim, 1);  // every thread has read it
            if (ctid == 0) tile_fx_store<NCW>(gs.red, p.tile_fx + 2 * tile);
            Ts64 a64{s_ts, base};
            tile_intervals<KIND>(p, sm, stage, a64, s_w, tile, (int64_t)INT64_MAX, cx, ctid);
            consumer_sync(g);
        }
        if (ctid == 0) {  // the group's stage reads / term writes before the producer's next bulk copy
            fence_proxy_async();
            mbar_arrive(&sm.empty[stage]);
        }
    }
}

// ------------------------------------------------ K2x exact-sum tile kernel
// DW_SUM_EXACT (every interval = the exact sum of its pieces rounded to
// 2^-40 W*us, rounded once).  Same producer as K2, with a shorter window halo
// (XHALO pieces: longer intervals take K4) so the ring holds XSTAGES stages:
// every consumer group holds one stage while it works, and the ring keeps
// XSTAGES - GROUPS tiles in flight ahead of them.  Per tile a consumer group:
//   pass B  one thread per XPER consecutive pieces of the window: the window's
//           32-bit relative timestamps, each piece's term and its fixed-point
//           value q (two instructions for |term| < 2^23 W*us), the thread's
//           share of the exact tile sum, and a warp scan of the q's (mod 2^64);
//   (group barrier)
//           the exclusive window prefix P[r] = sum of q over pieces < r, stored
//           into the stage's timestamp slots (mod 2^64);
//   (group barrier)
//   items   one thread per interval: locate its first piece and piece count
//           (the phase-1 search), its two edge pieces, and
//           q(first) + (P[s + cnt] - P[s]) + q(last) -- O(1) whatever the
//           length.  The modular difference is exact whenever the interval's
//           true sum is below 2^63 units; the bound (hi - lo) * max|w| <= 8e6
//           W*us guarantees it (|v| <= max|w| for every value the pieces use),
//           and intervals beyond the bound or XHALO pieces go to K4, which
//           sums the same pieces in int128.
// Each warp releases the stage on its own (empty barrier count = NCW): no
// barrier at the end of a tile; the 32-bit timestamps are double buffered.
#ifndef DW_XHALO
#define DW_XHALO 64
#endif
#ifndef DW_XSTAGES
#define DW_XSTAGES 8
#endif
constexpr int XHALO = DW_XHALO;                          // window halo = piece cap of the exact kernel
constexpr int XSTAGES = DW_XSTAGES;
constexpr int WINX = TILE + XHALO + 6;
constexpr int XPER = (((WINX + ATTR_THREADS - 1) / ATTR_THREADS) + 1) & ~1;  // pieces per thread in pass B (even)
static_assert(XPER % 2 == 0 && TILE % 2 == 0, "pass B's 16-byte shared-memory accesses need even XPER");
constexpr double X_BOUND = 8.0e6;  // W*us: |sum of an interval's q| < 2^63 below it
using TileSmemX = TileSmemT<XSTAGES, WINX>;
static_assert(GROUPS < XSTAGES, "claims in flight must span fewer positions than the ring");

// Per-set item descriptor of one tile (group smem, double buffered by tile
// parity): item v of set j (v in [c_j, c_{j+1}): the tile's items of all sets
// concatenated) is interval kq + v; its [start, end) sits at stage slot v + sx
// when v < lim; its joules go to out[v] (out pre-offset by kq; perm: the set
// was sorted on the device, so results scatter through p.perm).
struct __align__(16) SetDescX {
    double *out;
    int64_t kq;
    int sx, lim, pool, flags;  // flags: 1 check sorted, 2 perm
};

struct __align__(16) GroupSmemX {
    uint32_t ts32[2][WINX];
    SetDescX desc[2][DW_MAX_SETS];
    unsigned long long wtot[NCW];    // warp totals of the q scan (mod 2^64)
    long long red[2][NCW][2];        // warp shares of the exact tile sum (by tile parity)
    uint32_t wmax[NCW];              // warp max of the high word of |w|
    int next_it[2];                  // claimed next tile, by parity (claimed during pass B)
};

// Interior value v(x) of a linear signal at window slot r (energy.py:115-124:
// w[r-1] + 1.0 * (w[r] - w[r-1]); the signal's first / last sample hold w0 /
// wl; rz0 / rzS are their window slots or out of range).
__device__ __forceinline__ double lin_v(const double *w, int r, int rz0, int rzS, double w0, double wl) {
    const double wa = w[r > 0 ? r - 1 : 0];
    const double v = __dadd_rn(wa, __dsub_rn(w[r], wa));
    return r == rz0 ? w0 : (r == rzS ? wl : v);
}

__device__ __forceinline__ uint32_t abs_hi(double x) { return (uint32_t)__double2hiint(x) & 0x7FFFFFFFu; }

// Exact per-interval sum with O(1) work per interval.  Per tile a consumer
// group:
//   pass B  one thread per XPER consecutive pieces from the tile's first
//           sample r0: 32-bit relative timestamps (for the searches), each
//           piece's doubled term t2 = (v_r + v_r+1) * width (linear) or
//           2 * w_r * width (step) and q = rni(t2 * 2^39) -- bit for bit
//           q40(term), as 0.5 * x is exact -- the thread's running sum of q
//           (mod 2^64), its exact share of the tile sum (int64 for pieces
//           below 2^20 W*us; int128 term by term otherwise) and max |w|.
//           Threads whose pieces are all interior, in range and narrow take
//           a 32-bit body with no per-piece conditions.
//   (group barrier)
//           the exclusive window prefix P[r] = sum of q over pieces < r (mod
//           2^64) into the stage's timestamp slots;
//   (group barrier)
//   items   one thread per interval: its first piece a and last piece b by
//           guessed search, the two edge pieces (interpolated endpoint values,
//           exact divisions) and q(F0) + (P[b] - P[a+1]) + q(L).  The modular
//           difference is exact: (hi - lo) * max|w| <= X_BOUND W*us bounds the
//           interval's sum below 2^63 units and every piece inside it below
//           2^23 W*us.  Longer or larger intervals go to K4 (int128 there).
// Every warp releases the stage on its own.
template <int KIND>
#ifdef DW_X_MAXNREG
__global__ void __maxnreg__(DW_X_MAXNREG) attribute_exact_kernel(AttrParams p) {
#else
__global__ void __launch_bounds__(KTHREADS, 1) attribute_exact_kernel(AttrParams p) {
#endif
    extern __shared__ __align__(128) unsigned char smem_raw[];
    TileSmemX &sm = *reinterpret_cast<TileSmemX *>(smem_raw);
    GroupSmemX *groups =
        reinterpret_cast<GroupSmemX *>(smem_raw + ((sizeof(TileSmemX) + 15) & ~(size_t)15));
    const int tid = threadIdx.x;
    if ((int64_t)blockIdx.x >= p.ntiles) return;

    const int64_t S = p.S;
    TileCtx cx;
    cx.ts0 = __ldg(p.ts);
    cx.tsl = __ldg(p.ts + S - 1);
    cx.w0 = __ldg(p.w);
    cx.wl = __ldg(p.w + S - 1);
    cx.span_lo = cx.ts0;
    cx.span_hi = KIND == DW_SIGNAL_STEP ? p.span_hi : cx.tsl;
    const int64_t nterms = KIND == DW_SIGNAL_STEP ? S : S - 1;

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < XSTAGES; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], NCW);  // one arrival per consumer warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < GROUPS) groups[tid].next_it[0] = tid;
    if (tid == 0) sm.claim = GROUPS;
    __syncthreads();

    if (tid >= GROUPS * ATTR_THREADS) {
        producer<TileSmemX, XHALO>(p, sm, cx.span_hi, (tid - GROUPS * ATTR_THREADS) >> 5);
        return;
    }
    const int g = tid / ATTR_THREADS;
    const int ctid = tid - g * ATTR_THREADS;
    const int lane = ctid & 31, warp = ctid >> 5;
    GroupSmemX &gs = groups[g];
    int par = 0;
    for (;; par ^= 1) {
        const int it = gs.next_it[par];
        const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
        if (tile >= p.ntiles) break;
        const int stage = it % XSTAGES;
        mbar_wait(&sm.full[stage], (uint32_t)((it / XSTAGES) & 1));
#ifdef DW_SKIP_CONSUMERS
        consumer_sync(g);
        if (ctid == 0) gs.next_it[par ^ 1] = atomicAdd(&sm.claim, 1);
        consumer_sync(g);
        if (lane == 0) mbar_arrive(&sm.empty[stage]);
        continue;
#endif
        const StageMeta &M = sm.meta[stage];
        const int64_t wb = M.wb;
        const int cnt = M.cnt;
        int64_t *s_ts = sm.ts[stage];
        const double *s_w = sm.w[stage];
        const int64_t base = s_ts[0];
        const int last = (KIND == DW_SIGNAL_STEP && wb + cnt == S) ? cnt : cnt - 1;  // last timestamp slot
        const bool wide = (s_ts[last] - base) >= (int64_t)0xFFFFFFF0LL;
        const int64_t t0g = tile * TILE;
        const int r0 = (int)(t0g - wb);
        const int r1 = (int)((t0g + TILE < S ? t0g + TILE : S) - wb);
        const int e1 = (int)((t0g + TILE < nterms ? t0g + TILE : nterms) - wb);
        const int rz0 = wb == 0 ? 0 : -1000;
        const int rzS = (S - 1 - wb) < (int64_t)WINX ? (int)(S - 1 - wb) : -1000;
        {
            const int64_t dt = s_ts[r1 < last ? r1 : last] - s_ts[r0];
            cx.scale = dt > 0 ? __fdividef((float)(r1 - r0), (float)dt) : 0.0f;
        }
        uint32_t *ts32 = gs.ts32[par];
        if (ctid < DW_MAX_SETS) {  // this tile's set descriptors
            const int j = ctid;
            SetDescX d;
            d.kq = M.f0[j] - M.c[j];
            const bool perm = j < p.nsets && p.perm[j] != nullptr;
            d.out = j < p.nsets && !perm ? p.out[j] + d.kq : nullptr;
            d.sx = (int)(M.pool[j] - M.a0[j] + d.kq);
            d.lim = (int)(M.a0[j] + M.copied[j] - d.kq);
            d.pool = M.pool[j];
            d.flags = (j < p.nsets && p.check_sorted[j] ? 1 : 0) | (perm ? 2 : 0);
            gs.desc[par][j] = d;
        }

        // the group's next tile, claimed early (read after this tile's barriers)
#ifndef DW_CLAIM_T
#define DW_CLAIM_T 32
#endif
#ifndef DW_TSUM_T
#define DW_TSUM_T 32
#endif
        if (ctid == DW_CLAIM_T) gs.next_it[par ^ 1] = atomicAdd(&sm.claim, 1);
        // ---- pass B: pieces rb .. rb + XPER - 1 (r < last)
        const int rb = r0 + ctid * XPER;
        long long q[XPER];
        unsigned long long run = 0;
        long long tin = 0;    // exact share of the tile sum (pieces [r0, e1)), int64 part
        i128 tbig = 0;        // ... and its int128 part (huge pieces)
        uint32_t hmax = 0;
        bool big = false, bad = false;
        const bool fastb = !wide && rb + XPER <= last && rb + XPER < cnt && !(rzS > rb && rzS <= rb + XPER) &&
                           (rb + XPER <= e1 || rb >= e1);
        if (fastb) {
            // the thread's XPER + 1 timestamps and watts (and w[rb - 1] for
            // v(rb)) as 16-byte loads: rb is even, so every pair is aligned,
            // and lanes XPER * 8 bytes apart hit distinct banks per quarter warp
            const uint32_t b32 = (uint32_t)base;
            int64_t tv[XPER + 2];
            double wv[XPER + 4];  // wv[i] = w[rb - 2 + i]
#pragma unroll
            for (int i = 0; i < XPER; i += 2) {
                const longlong2 t2v = *reinterpret_cast<const longlong2 *>(s_ts + rb + i);
                tv[i] = t2v.x;
                tv[i + 1] = t2v.y;
            }
            tv[XPER] = s_ts[rb + XPER];
#pragma unroll
            for (int i = (KIND == DW_SIGNAL_LINEAR ? 0 : 2); i < XPER + 2; i += 2) {
                const double2 w2v = *reinterpret_cast<const double2 *>(s_w + rb - 2 + i);
                wv[i] = w2v.x;
                wv[i + 1] = w2v.y;
            }
            wv[XPER + 2] = s_w[rb + XPER];
            int64_t t0 = tv[0];
            double wcur = wv[2];
            double vcur = 0.0;
            if (KIND == DW_SIGNAL_LINEAR)
                vcur = rb == rz0 ? cx.w0 : (rb == rzS ? cx.wl : __dadd_rn(wv[1], __dsub_rn(wcur, wv[1])));
            hmax = abs_hi(wcur);
#pragma unroll
            for (int i = 0; i < XPER; i += 2)  // 32-bit window timestamps, two per store
                *reinterpret_cast<uint2 *>(ts32 + rb + i) =
                    make_uint2((uint32_t)tv[i] - b32, (uint32_t)tv[i + 1] - b32);
#pragma unroll
            for (int i = 0; i < XPER; ++i) {
                const int64_t t1 = tv[i + 1];
                bad |= t1 <= t0;
                const double wd = (double)((uint32_t)t1 - (uint32_t)t0);
                const double wnext = wv[i + 3];
                double t2;
                if (KIND == DW_SIGNAL_STEP) {
                    t2 = __dmul_rn(__dadd_rn(wcur, wcur), wd);
                } else {
                    const double vnext = __dadd_rn(wcur, __dsub_rn(wnext, wcur));
                    t2 = __dmul_rn(__dadd_rn(vcur, vnext), wd);
                    vcur = vnext;
                }
                hmax = max(hmax, abs_hi(wnext));
                wcur = wnext;
                big |= !(fabs(t2) < 2097152.0);  // 2^21: |q| < 2^60, the share of XPER pieces fits int64
                q[i] = __double2ll_rn(__dmul_rn(t2, 549755813888.0));  // * 2^39
                run += (unsigned long long)q[i];
                t0 = t1;
            }
            if (rb < e1) tin = (long long)run;
        } else {
#pragma unroll
            for (int i = 0; i < XPER; ++i) {
                const int r = rb + i;
                q[i] = 0;
                if (!wide && r <= last) ts32[r] = (uint32_t)(s_ts[r] - base);
                if (r < last) {
                    const int64_t t0 = s_ts[r], t1 = s_ts[r + 1];
                    bad |= t1 <= t0;
                    const int64_t width = t1 - t0;
                    double t2;
                    if (KIND == DW_SIGNAL_STEP) {
                        const double wv = s_w[r];
                        hmax = max(hmax, abs_hi(wv));
                        t2 = __dmul_rn(__dadd_rn(wv, wv), (double)width);
                    } else {
                        hmax = max(hmax, max(abs_hi(s_w[r]), abs_hi(s_w[r + 1])));
                        t2 = __dmul_rn(__dadd_rn(lin_v(s_w, r, rz0, rzS, cx.w0, cx.wl),
                                                 lin_v(s_w, r + 1, rz0, rzS, cx.w0, cx.wl)), (double)width);
                    }
                    q[i] = __double2ll_rn(__dmul_rn(t2, 549755813888.0));
                    run += (unsigned long long)q[i];
                    if (r < e1) tbig += q40(__dmul_rn(t2, 0.5));
                }
            }
        }
        if (big) {  // a piece of 2^20 W*us or more: this thread's share term by term in int128
            tin = 0;
            for (int i = 0; i < XPER; ++i) {
                const int r = rb + i;
                if (r >= e1) break;
                const double wd = (double)(s_ts[r + 1] - s_ts[r]);
                const double term = KIND == DW_SIGNAL_STEP
                                        ? __dmul_rn(s_w[r], wd)
                                        : __dmul_rn(__dmul_rn(0.5, __dadd_rn(lin_v(s_w, r, rz0, rzS, cx.w0, cx.wl),
                                                                             lin_v(s_w, r + 1, rz0, rzS, cx.w0, cx.wl))),
                                                    wd);
                tbig += q40(term);
            }
        }
        // warp inclusive scan of the per-thread sums (mod 2^64)
        unsigned long long inc = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const uint32_t wm = __reduce_max_sync(0xffffffffu, hmax);
        // the warp's exact share of the tile sum: int64 shares as three 21-bit
        // limb sums (32-bit reductions), int128 spills (rare) by shuffles
        {
            const int l0 = __reduce_add_sync(0xffffffffu, (int)(tin & 0x1FFFFF));
            const int l1 = __reduce_add_sync(0xffffffffu, (int)((tin >> 21) & 0x1FFFFF));
            const int l2 = __reduce_add_sync(0xffffffffu, (int)(tin >> 42));
            i128 spill = 0;
            if (__any_sync(0xffffffffu, tbig != 0)) spill = warp_sum_i128(tbig);
            if (lane == 0) {
                const i128 t = (i128)l0 + ((i128)l1 << 21) + ((i128)l2 << 42) + spill;
                const I128Parts pp = split(t);
                gs.red[par][warp][0] = (long long)pp.lo;
                gs.red[par][warp][1] = (long long)pp.hi;
                gs.wmax[warp] = wm;
            }
        }
        if (lane == 31) gs.wtot[warp] = inc;
        if (p.validate_order && bad) {  // strictly increasing power timestamps: the first offender
            for (int i = 0; i < XPER; ++i) {
                const int r = rb + i;
                if (r < r1 && wb + r + 1 < S && r < last && s_ts[r + 1] <= s_ts[r])
                    atomic_min_index(&p.st->order_index, wb + r);
            }
        }
        consumer_sync(g);
        // ---- the exclusive window prefix into the stage's timestamp slots
        uint32_t wmx_hi = 0;
        {
            unsigned long long pre = inc - run;
#pragma unroll
            for (int k = 0; k < NCW; ++k) {
                if (k < warp) pre += gs.wtot[k];
                wmx_hi = max(wmx_hi, gs.wmax[k]);
            }
            unsigned long long *P = reinterpret_cast<unsigned long long *>(s_ts);
            if (fastb) {
#pragma unroll
                for (int i = 0; i < XPER; i += 2) {  // 16-byte stores (rb even)
                    const unsigned long long p1 = pre + (unsigned long long)q[i];
                    *reinterpret_cast<ulonglong2 *>(P + rb + i) = make_ulonglong2(pre, p1);
                    pre = p1 + (unsigned long long)q[i + 1];
                }
            } else {
#pragma unroll
                for (int i = 0; i < XPER; ++i) {
                    if (rb + i <= last) P[rb + i] = pre;
                    pre += (unsigned long long)q[i];
                }
            }
        }
        consumer_sync(g);
        const unsigned long long *P = reinterpret_cast<const unsigned long long *>(s_ts);
        if (ctid == DW_TSUM_T) {  // the exact tile sum (its shares are double buffered)
            i128 t = 0;
#pragma unroll
            for (int k = 0; k < NCW; ++k) t += join((uint64_t)gs.red[par][k][0], (uint64_t)gs.red[par][k][1]);
            const I128Parts pp = split(t);
            p.tile_fx[2 * tile] = pp.lo;
            p.tile_fx[2 * tile + 1] = pp.hi;
        }
        // max |w| over the window, rounded up (NaN / inf: every bound test fails)
        const double wmx = __hiloint2double((int)(wmx_hi + 1u), 0);

        // ---- items: one interval per thread
        const int total = (int)M.c[DW_MAX_SETS];
        const int c1 = (int)M.c[1], c2 = (int)M.c[2], c3 = (int)M.c[3];
        const int64_t *s_lo = sm.iv_lo[stage], *s_hi = sm.iv_hi[stage];
        const SetDescX *dsc = gs.desc[par];
        const bool first_tile = wb == 0;
        const uint32_t tr0 = ts32[r0];
#ifdef DW_X_NO_ITEMS
        if (total >= 0) { __syncwarp(); if (lane == 0) mbar_arrive(&sm.empty[stage]); continue; }
#endif
#ifndef DW_ITEM_SPREAD
#define DW_ITEM_SPREAD 1
#endif
        // the last, partial round of items spread over DW_ITEM_SPREAD warps
        // (1: lanes of the first warps, as full rounds)
        constexpr int SPK = DW_ITEM_SPREAD;
        const int vlast = ctid / (32 * SPK) * (32 * SPK) + lane * SPK + warp % SPK;
        const int tfull = total - total % ATTR_THREADS;
        for (int v0 = 0; v0 < total; v0 += ATTR_THREADS) {
            const int v = v0 + (SPK > 1 && v0 == tfull ? vlast : ctid);
            if (v >= total) break;
            const int j = (v >= c1) + (v >= c2) + (v >= c3);
            const SetDescX d = dsc[j];
            const int slot = v + d.sx;
            int64_t glo, ghi;
            const bool staged = v < d.lim;
            if (staged) {
                glo = s_lo[slot];
                ghi = s_hi[slot];
            } else {  // beyond the staged pool (rare)
                glo = __ldg(p.start[j] + d.kq + v);
                ghi = __ldg(p.end[j] + d.kq + v);
            }
            if (d.flags & 1) {  // a set flagged sorted must be sorted by start
                const int64_t k = d.kq + v;
                const int64_t prev = (staged && slot > d.pool) ? s_lo[slot - 1]
                                                               : (k > 0 ? __ldg(p.start[j] + k - 1) : glo);
                if (prev > glo) atomic_min_index(&p.st->unsorted_index[j], k);
            }
            if (ghi < glo || ghi > cx.span_hi || (first_tile && glo < cx.span_lo)) {
                report_bad(p, j, d.kq + v);
                continue;
            }
            const int64_t dh = ghi - base;
            bool ok = !wide && dh <= (int64_t)0xFFFFFFFFLL && __dmul_rn((double)(ghi - glo), wmx) <= X_BOUND;
            double J = 0.0;
            if (ok) {
                const uint32_t lo = (uint32_t)glo - (uint32_t)base;
                const uint32_t hi = (uint32_t)dh;
                const int a = find_le4(ts32, r0, r1, lo, tr0, r0, cx.scale);
                const uint32_t ta = ts32[a], ta1 = ts32[a + 1];
                const int lim = min(a + XHALO + 1, cnt);
                double F2, L2;
                int b;
                bool one;
                if (KIND == DW_SIGNAL_STEP) {
                    // pieces: none (hi == lo); w[a]*(hi-lo) inside one segment;
                    // else first partial + whole interior + last partial segment
                    b = hi > lo ? find_le4(ts32, a, lim, hi - 1, ta, a, cx.scale) : a;
                    ok = b - a < XHALO;  // segments b - a + 1 <= XHALO
                    const double wa = s_w[a];
                    one = b == a;
                    F2 = __dmul_rn(__dadd_rn(wa, wa), (double)((one ? hi : ta1) - lo));
                    const double wbv = s_w[b];
                    L2 = __dmul_rn(__dadd_rn(wbv, wbv), (double)(hi - ts32[b]));
                } else {
                    // pieces [lo, ts] .. [ts, hi] (energy.py:108-130); b = last sample < hi
                    b = ta < hi ? find_le4(ts32, a, lim, hi - 1, ta, a, cx.scale) : a - 1;
                    const int m = b - a;  // -1 only when hi == lo == ts[a]
                    ok = m < XHALO;       // pieces m + 1 <= XHALO
                    const int il = ta == lo && a > 0 ? a - 1 : a;  // first bracketing pair (energy.py:115-124)
                    const double wl0 = s_w[il], wl1 = s_w[il + 1];
                    const uint32_t tl0 = ts32[il];
                    const double vlo_i = __dadd_rn(wl0, __dmul_rn(div_u32(lo - tl0, ts32[il + 1] - tl0), __dsub_rn(wl1, wl0)));
                    const double vlo = glo <= cx.ts0 ? cx.w0 : (glo >= cx.tsl ? cx.wl : vlo_i);
                    const double wh0 = s_w[b], wh1 = s_w[b + 1];
                    const uint32_t th0 = ts32[b];
                    const double vhi_i = __dadd_rn(wh0, __dmul_rn(div_u32(hi - th0, ts32[b + 1] - th0), __dsub_rn(wh1, wh0)));
                    const double vhi = ghi <= cx.ts0 ? cx.w0 : (ghi >= cx.tsl ? cx.wl : vhi_i);
                    one = m <= 0;  // one piece [lo, hi]
                    const double wa = s_w[a];
                    const double vn = one ? vhi : __dadd_rn(wa, __dsub_rn(s_w[a + 1], wa));
                    F2 = __dmul_rn(__dadd_rn(vlo, vn), (double)((one ? hi : ta1) - lo));
                    const double wbm = s_w[b > 0 ? b - 1 : 0];
                    L2 = __dmul_rn(__dadd_rn(__dadd_rn(wbm, __dsub_rn(wh0, wbm)), vhi), (double)(hi - th0));
                }
                // |F2|, |L2| < 2^24 follow from the bound: rni is exact in int64
                long long tq = __double2ll_rn(__dmul_rn(F2, 549755813888.0));
                if (!one) tq += __double2ll_rn(__dmul_rn(L2, 549755813888.0)) + (long long)(P[b] - P[a + 1]);
                J = div_1e6(__dmul_rn((double)tq, 9.094947017729282379150390625e-13));  // * 2^-40
            }
            if (!ok) {
                push_long(p, j, d.kq + v);
            } else if (!(d.flags & 2)) {
                d.out[v] = J;
            } else {
                p.out[j][__ldg(p.perm[j] + d.kq + v)] = J;
            }
        }
        // release the stage: every lane's reads (and its pass-B writes of P
        // into the stage) ordered before the producer's next bulk copy into it
        // -- a generic->async proxy fence per lane, warp sync, then the
        // release-arrive the producer acquires
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[stage]);
    }
}

// ------------------------------------------------------------ K3 tile scan
// exact int128 exclusive prefix of q(tile_sum) over tiles: block partials,
// one-block scan of partials, block rescan (coalesced, 3 small launches)
constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_PER_THREAD = 4;
constexpr int SCAN_CHUNK = SCAN_THREADS * SCAN_PER_THREAD;

__device__ __forceinline__ i128 block_exclusive_scan(i128 v, i128 &block_total) {
    __shared__ unsigned long long s[SCAN_THREADS / 32][2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    i128 x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        I128Parts q = split(x);
        uint64_t lo = __shfl_up_sync(0xffffffffu, q.lo, o);
        uint64_t hi = __shfl_up_sync(0xffffffffu, q.hi, o);
        if (lane >= o) x += join(lo, hi);
    }
    if (lane == 31) {
        I128Parts q = split(x);
        s[warp][0] = q.lo;
        s[warp][1] = q.hi;
    }
    __syncthreads();
    if (warp == 0) {
        i128 y = lane < SCAN_THREADS / 32 ? join(s[lane][0], s[lane][1]) : (i128)0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            I128Parts q = split(y);
            uint64_t lo = __shfl_up_sync(0xffffffffu, q.lo, o);
            uint64_t hi = __shfl_up_sync(0xffffffffu, q.hi, o);
            if (lane >= o) y += join(lo, hi);
        }
        I128Parts q = split(y);
        s[lane][0] = q.lo;
        s[lane][1] = q.hi;
    }
    __syncthreads();
    block_total = join(s[SCAN_THREADS / 32 - 1][0], s[SCAN_THREADS / 32 - 1][1]);
    i128 warp_base = warp ? join(s[warp - 1][0], s[warp - 1][1]) : (i128)0;
    __syncthreads();
    return warp_base + x - v;
}

__device__ __forceinline__ i128 thread_chunk(const AttrParams &p, int64_t b0, i128 *vals) {
    i128 sum = 0;
#pragma unroll
    for (int k = 0; k < SCAN_PER_THREAD; ++k) {
        int64_t b = b0 + k;
        i128 v = b < p.ntiles ? join(p.tile_fx[2 * b], p.tile_fx[2 * b + 1]) : (i128)0;
        if (vals) vals[k] = v;
        sum += v;
    }
    return sum;
}

__global__ void __launch_bounds__(SCAN_THREADS) scan_partials_kernel(AttrParams p) {
    int64_t b0 = (int64_t)blockIdx.x * SCAN_CHUNK + threadIdx.x * SCAN_PER_THREAD;
    i128 sum = thread_chunk(p, b0, nullptr);
    i128 total;
    block_exclusive_scan(sum, total);
    if (threadIdx.x == 0) {
        I128Parts q = split(total);
        p.scan_part[2 * blockIdx.x] = q.lo;
        p.scan_part[2 * blockIdx.x + 1] = q.hi;
    }
}

__global__ void __launch_bounds__(SCAN_THREADS) scan_top_kernel(AttrParams p, int64_t nblocks) {
    // exclusive scan of block partials, in place (nblocks <= a few thousand)
    __shared__ unsigned long long carry[2];
    if (threadIdx.x == 0) { carry[0] = 0; carry[1] = 0; }
    __syncthreads();
    for (int64_t c = 0; c < nblocks; c += SCAN_THREADS) {
        int64_t b = c + threadIdx.x;
        i128 v = b < nblocks ? join(p.scan_part[2 * b], p.scan_part[2 * b + 1]) : (i128)0;
        i128 total;
        i128 ex = block_exclusive_scan(v, total);
        i128 base = join(carry[0], carry[1]);
        if (b < nblocks) {
            I128Parts q = split(base + ex);
            p.scan_part[2 * b] = q.lo;
            p.scan_part[2 * b + 1] = q.hi;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            I128Parts q = split(base + total);
            carry[0] = q.lo;
            carry[1] = q.hi;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {  // grand total at prefix[ntiles]
        p.prefix[2 * p.ntiles] = carry[0];
        p.prefix[2 * p.ntiles + 1] = carry[1];
    }
}

__global__ void __launch_bounds__(SCAN_THREADS) scan_apply_kernel(AttrParams p) {
    int64_t b0 = (int64_t)blockIdx.x * SCAN_CHUNK + threadIdx.x * SCAN_PER_THREAD;
    i128 vals[SCAN_PER_THREAD];
    i128 sum = thread_chunk(p, b0, vals);
    i128 total;
    i128 run = block_exclusive_scan(sum, total) +
               join(p.scan_part[2 * blockIdx.x], p.scan_part[2 * blockIdx.x + 1]);
#pragma unroll
    for (int k = 0; k < SCAN_PER_THREAD; ++k) {
        int64_t b = b0 + k;
        if (b < p.ntiles) {
            I128Parts q = split(run);
            p.prefix[2 * b] = q.lo;
            p.prefix[2 * b + 1] = q.hi;
        }
        run += vals[k];
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

// exact sum of terms [j0, j1] (inclusive): partial tiles term by term, whole
// tiles through the int128 prefix of the exact tile sums; whole warp participates
template <int KIND>
__device__ i128 range_sum(const AttrParams &p, int64_t j0, int64_t j1) {
    const int lane = threadIdx.x & 31;
    if (j1 < j0) return 0;
    auto span_sum = [&](int64_t a, int64_t b) -> i128 {
        i128 acc = 0;
        for (int64_t i = a + lane; i <= b; i += 32) acc += q40(term_global<KIND>(p, i));
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
            if (hi <= lo || a >= b) {  // no piece, or one piece inside segment a (exact mode's wide windows)
                acc = (lane == 0 && hi > lo) ? q_term(__dmul_rn(W(a), (double)(hi - lo))) : (i128)0;
            } else {
                acc = range_sum<KIND>(p, a + 1, b - 1);
                if (lane == 0) {
                    acc += q_term(__dmul_rn(W(a), (double)(TS(a + 1) - lo)));
                    acc += q_term(__dmul_rn(W(b), (double)(min(TS(b + 1), hi) - TS(b))));
                }
            }
        } else {
            int64_t first = upper_bound_g(p.ts, S, lo);
            int64_t last = lower_bound_g(p.ts, S, hi);
            if (last <= first) {  // no sample strictly inside: the one piece [lo, hi]
                acc = 0;
                if (lane == 0) {
                    const double vlo = lin_value_at(lo, (first > 0 && TS(first - 1) == lo) ? first - 1 : first, TS(0),
                                                    TS(S - 1), W(0), W(S - 1), TS, W);
                    const double vh = lin_value_at(hi, last, TS(0), TS(S - 1), W(0), W(S - 1), TS, W);
                    acc = q_term(lin_piece(vlo, vh, hi - lo));
                }
            } else {
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
        }
        if (lane == 0) {
            int64_t oidx = p.perm[j] ? __ldg(p.perm[j] + k) : k;
            p.out[j][oidx] = term_fx_to_joules(acc);
        }
    }
}

// --------------------------------------------- K7 time-window partials
// One rank of a time-window-sharded trace holds the samples of
// its owned pieces [P0, P1) (global indices) plus halos; its tile grid is the
// global one (g_off, the global index of local sample 0, is a multiple of
// DW_TILE).  For each listed interval -- an interval longer than DW_DIRECT_MAX
// pieces that crosses window edges -- this computes the exact fixed-point
// contribution of the pieces it owns, with the same decomposition as
// long_intervals_kernel (edge pieces, partial tiles term by term, whole tiles
// through the tile prefix), so the sum over ranks equals the one-GPU value
// bit for bit.  Sample values use the GLOBAL first / last sample rules.
struct WindowParams {
    int64_t g_off, S_global, P0, P1;
    int64_t ts0_g, tsl_g;  // global first / last sample time
    double w0_g, wl_g;     // and watts
};

template <int KIND>
__global__ void __launch_bounds__(256) window_partials_kernel(AttrParams p, WindowParams wp, const int64_t *blo,
                                                             const int64_t *bhi, int64_t nb,
                                                             unsigned long long *part) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
    const int64_t S = p.S, g = wp.g_off;
    auto TS = [&](int64_t i) -> int64_t { return i < S ? __ldg(p.ts + i) : p.span_hi; };
    auto W = [&](int64_t i) -> double { return __ldg(p.w + i); };
    auto VS = [&](int64_t j) -> double {  // v(ts[j]) with the global boundary rules
        if (j + g == 0 || j + g == wp.S_global - 1) return W(j);
        const double wa = W(j - 1);
        return __dadd_rn(wa, __dsub_rn(W(j), wa));
    };
    auto own = [&](int64_t jg) -> bool { return jg >= wp.P0 && jg < wp.P1; };
    // owned share of range_sum over GLOBAL pieces [j0g, j1g], with the one-GPU
    // decomposition: its first and last tiles term by term, the tiles between
    // through their tile sums (each tile is owned by exactly one rank)
    auto termwise = [&](int64_t a, int64_t b) -> i128 {  // global, clipped to the owned pieces
        a = max(a, wp.P0);
        b = min(b, wp.P1 - 1);
        i128 acc = 0;
        for (int64_t i = a + lane; i <= b; i += 32) acc += q_term(term_global<KIND>(p, i - g));
        return warp_sum_i128(acc);
    };
    auto clipped = [&](int64_t j0g, int64_t j1g) -> i128 {
        if (j1g < j0g) return (i128)0;
        const int64_t ta = j0g / TILE, tb = j1g / TILE;
        if (ta == tb) return termwise(j0g, j1g);
        i128 s = termwise(j0g, (ta + 1) * TILE - 1) + termwise(tb * TILE, j1g);
        const int64_t w0 = max(ta + 1, wp.P0 / TILE), w1 = min(tb, (wp.P1 + TILE - 1) / TILE);  // owned whole tiles
        if (w1 > w0) {
            const int64_t l0 = w0 - g / TILE, l1 = w1 - g / TILE;
            s += join(p.prefix[2 * l1], p.prefix[2 * l1 + 1]) - join(p.prefix[2 * l0], p.prefix[2 * l0 + 1]);
        }
        return s;
    };
    for (int64_t e = warp; e < nb; e += nwarps) {
        const int64_t lo = blo[e], hi = bhi[e];
        i128 acc;
        if (KIND == DW_SIGNAL_STEP) {
            const int64_t al = upper_bound_g(p.ts, S, lo) - 1;     // segment holding lo (-1: before the data)
            const int64_t bl = hi > TS(S) ? S : lower_bound_g(p.ts, S, hi) - 1;  // S: past the data
            const int64_t ag = al < 0 ? g - 1 : al + g, bg = bl + g;
            acc = clipped(ag + 1, bg - 1);
            if (lane == 0) {
                if (al >= 0 && own(ag)) acc += q_term(__dmul_rn(W(al), (double)(TS(al + 1) - lo)));
                if (bl < S && own(bg)) acc += q_term(__dmul_rn(W(bl), (double)(min(TS(bl + 1), hi) - TS(bl))));
            }
        } else {
            const int64_t fl = upper_bound_g(p.ts, S, lo);          // first sample > lo (0: at or before the data)
            const int64_t ll = hi > TS(S - 1) ? S + 1 : lower_bound_g(p.ts, S, hi);  // first sample >= hi
            const int64_t fg = fl + g, lg = ll + g;
            acc = clipped(fg, lg - 2);
            if (lane == 0) {
                if (fl > 0 && own(fg - 1)) {  // left edge piece [lo, ts[first]]
                    const int64_t i = (TS(fl - 1) == lo && fl - 1 > 0) ? fl - 2 : fl - 1;  // first bracketing pair
                    double vlo;
                    if (lo <= wp.ts0_g) vlo = wp.w0_g;
                    else if (lo >= wp.tsl_g) vlo = wp.wl_g;
                    else {
                        const double wa = W(i);
                        const double fr = __ddiv_rn((double)(lo - TS(i)), (double)(TS(i + 1) - TS(i)));
                        vlo = __dadd_rn(wa, __dmul_rn(fr, __dsub_rn(W(i + 1), wa)));
                    }
                    acc += q_term(lin_piece(vlo, VS(fl), TS(fl) - lo));
                }
                if (ll <= S && own(lg - 1)) {  // right edge piece [ts[last-1], hi]
                    const int64_t i = ll - 1;
                    double vh;
                    if (hi <= wp.ts0_g) vh = wp.w0_g;
                    else if (hi >= wp.tsl_g) vh = wp.wl_g;
                    else {
                        const double wa = W(i);
                        const double fr = __ddiv_rn((double)(hi - TS(i)), (double)(TS(i + 1) - TS(i)));
                        vh = __dadd_rn(wa, __dmul_rn(fr, __dsub_rn(W(i + 1), wa)));
                    }
                    acc += q_term(lin_piece(VS(i), vh, hi - TS(i)));
                }
            }
        }
        if (lane == 0) {
            const I128Parts pp = split(acc);
            part[2 * e] = pp.lo;
            part[2 * e + 1] = pp.hi;
        }
    }
}

// exact int128 sum of q(tile_sum) over local tiles [t0, t1) -> out[2]
__global__ void tile_range_kernel(AttrParams p, int64_t t0, int64_t t1, unsigned long long *out) {
    if (threadIdx.x != 0) return;
    const i128 v = join(p.prefix[2 * t1], p.prefix[2 * t1 + 1]) - join(p.prefix[2 * t0], p.prefix[2 * t0 + 1]);
    const I128Parts pp = split(v);
    out[0] = pp.lo;
    out[1] = pp.hi;
}

// ------------------------------------------------------- K5 sums / finalize
constexpr int SUM_THREADS = 512;
constexpr int SUM_BLOCKS = 1024;  // partial slots in the workspace
// Exact fixed-point sum (2^-64 J) with the last-block-done pattern.
__global__ void __launch_bounds__(SUM_THREADS) fx_sum_kernel(const double *x, int64_t n,
                                                             unsigned long long *partials,
                                                             unsigned int *done, double *out,
                                                             unsigned long long *out_fx = nullptr) {
    __shared__ unsigned long long red[SUM_THREADS / 32][2];
    __shared__ bool last;
    i128 acc = 0;
    constexpr int U = 8;  // loads in flight per thread
    const int64_t stride = (int64_t)gridDim.x * SUM_THREADS;
    for (int64_t i0 = blockIdx.x * (int64_t)SUM_THREADS + threadIdx.x; i0 < n; i0 += U * stride) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + (int64_t)u * stride;
            v[u] = i < n ? __ldcs(x + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += fx_joules(v[u]);
    }
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
    if (!last) return;
    // the last block sums the per-block partials with all its threads (L2
    // loads, independent), not one thread's chain of dependent round trips
    __threadfence();
    i128 part = 0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += SUM_THREADS)
        part += join(__ldcg(partials + 2 * b), __ldcg(partials + 2 * b + 1));
    part = warp_sum_i128(part);
    if ((threadIdx.x & 31) == 0) {
        I128Parts pp = split(part);
        red[threadIdx.x >> 5][0] = pp.lo;
        red[threadIdx.x >> 5][1] = pp.hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        i128 s = 0;
        for (int k = 0; k < SUM_THREADS / 32; ++k) s += join(red[k][0], red[k][1]);
        if (out) *out = fx_to_double(s, FX_JOULE_BITS);
        if (out_fx) {
            const I128Parts pp = split(s);
            out_fx[0] = pp.lo;
            out_fx[1] = pp.hi;
        }
        *done = 0;  // reusable
    }
}

// One resident wave: every block of the sum is on an SM at once (no tail
// wave), capped at SUM_BLOCKS partials.
static unsigned sum_grid(int64_t n) {
    static int per_sm = 0;
    if (!per_sm && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fx_sum_kernel, SUM_THREADS, 0) !=
                       cudaSuccess)
        per_sm = 1;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(SUM_BLOCKS, (int64_t)num_sms() * per_sm),
                                                            ceil_div(n, SUM_THREADS)));
}

// total over the whole span + idle (energy.py:318-324)
template <int KIND>
__global__ void ledger_finalize_kernel(AttrParams p, const double *op_total) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int64_t S = p.S;
    const int64_t nterms = KIND == DW_SIGNAL_STEP ? S : (S > 1 ? S - 1 : 1);
    double total;
    if (nterms <= DIRECT && p.sum_mode != DW_SUM_EXACT) {
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
    size_t status, first, tile_sum, prefix, scan_part, long_list, sum_partials, sum_done, sum_out;
    size_t pidx[DW_MAX_SETS];
    size_t sort_keys[DW_MAX_SETS], sort_perm[DW_MAX_SETS], sort_end[DW_MAX_SETS],
        sort_iota[DW_MAX_SETS];
    size_t cub_tmp, cub_bytes, total;
};


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
    L.tile_sum = off; off += align_up(16 * (size_t)(ntiles + 1));
    L.prefix = off; off += align_up(16 * (size_t)(ntiles + 2));
    L.scan_part = off; off += align_up(16 * (size_t)(ceil_div(ntiles, SCAN_CHUNK) + 1));
    L.long_list = off; off += align_up(8 * (size_t)(nint + 1));
    L.sum_partials = off; off += align_up(16 * (size_t)SUM_BLOCKS);
    L.sum_done = off; off += align_up(16);
    L.sum_out = off; off += align_up(16);
    for (int j = 0; j < nsets; ++j) {
        L.pidx[j] = off;
        off += align_up(8 * (size_t)(ceil_div(sizes[j], PIDX_STRIDE) + 1));
    }
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

// SMs the tile kernel may occupy (0: all).  Leaving a few free lets work on
// another stream (the join's pairing) run beside it: the tile kernel is a
// persistent one-CTA-per-SM kernel that otherwise fills the whole GPU.
static int g_attr_sms = 0;

struct WindowJob {  // dw_attribute_window: work after the tile kernel on the same tile prefix
    WindowParams wp;
    const int64_t *blo, *bhi;
    int64_t nb;
    unsigned long long *part;  // [2 nb]
    int64_t t0, t1;            // owned local tiles
    unsigned long long *tile_fx;  // [2]
};

static int attribute_impl(const dw_signal_t *sig, dw_interval_set_t *sets, int nsets,
                          void *ws, size_t ws_bytes, cudaStream_t stream, bool ledger,
                          dw_interval_set_t *ops_for_total, const WindowJob *wj = nullptr) {
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
    p.sum_mode = sig->sum_mode == DW_SUM_EXACT ? DW_SUM_EXACT : DW_SUM_REFERENCE;
    p.first = (const int64_t *)(base + L.first);
    p.tile_fx = (unsigned long long *)(base + L.tile_sum);
    p.scan_part = (unsigned long long *)(base + L.scan_part);
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
        PartIndex pix{};
        int64_t mmax = 0;
        for (int j = 0; j < nsets; ++j) {
            pix.p[j] = (int64_t *)(base + L.pidx[j]);
            mmax = std::max<int64_t>(mmax, ceil_div(p.n[j], PIDX_STRIDE));
        }
        if (mmax > 0) {
            partition_index_kernel<<<(unsigned)ceil_div(mmax, 256), 256, 0, stream>>>(p, pix, nsets);
            count_launch();
        }
        partition_kernel<<<(unsigned)ceil_div(nb, 256), 256, 0, stream>>>(p, pix);
        count_launch();
    }
    const size_t smem = ((sizeof(TileSmem) + 15) & ~(size_t)15) + GROUPS * sizeof(GroupSmem);
    const int sms = g_attr_sms > 0 && g_attr_sms < num_sms() ? g_attr_sms : num_sms();
    int grid = (int)std::min<int64_t>(p.ntiles, (int64_t)sms * CTAS_PER_SM);
    const size_t smem_x = ((sizeof(TileSmemX) + 15) & ~(size_t)15) + GROUPS * sizeof(GroupSmemX);
    timing_begin(stream);
    if (p.sum_mode == DW_SUM_EXACT) {
        if (sig->kind == DW_SIGNAL_STEP) {
            cudaFuncSetAttribute(attribute_exact_kernel<DW_SIGNAL_STEP>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_x);
            attribute_exact_kernel<DW_SIGNAL_STEP><<<grid, KTHREADS, smem_x, stream>>>(p);
        } else {
            cudaFuncSetAttribute(attribute_exact_kernel<DW_SIGNAL_LINEAR>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_x);
            attribute_exact_kernel<DW_SIGNAL_LINEAR><<<grid, KTHREADS, smem_x, stream>>>(p);
        }
    } else if (sig->kind == DW_SIGNAL_STEP) {
        cudaFuncSetAttribute(attribute_tiles_kernel<DW_SIGNAL_STEP>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attribute_tiles_kernel<DW_SIGNAL_STEP><<<grid, KTHREADS, smem, stream>>>(p);
    } else {
        cudaFuncSetAttribute(attribute_tiles_kernel<DW_SIGNAL_LINEAR>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attribute_tiles_kernel<DW_SIGNAL_LINEAR><<<grid, KTHREADS, smem, stream>>>(p);
    }
    timing_end(stream);
    count_launch();
    {
        const int64_t nblk = ceil_div(p.ntiles, SCAN_CHUNK);
        scan_partials_kernel<<<(unsigned)nblk, SCAN_THREADS, 0, stream>>>(p);
        scan_top_kernel<<<1, SCAN_THREADS, 0, stream>>>(p, nblk);
        scan_apply_kernel<<<(unsigned)nblk, SCAN_THREADS, 0, stream>>>(p);
        count_launch(3);
    }
    const int long_grid = num_sms() * 4;
    if (sig->kind == DW_SIGNAL_STEP)
        long_intervals_kernel<DW_SIGNAL_STEP><<<long_grid, 256, 0, stream>>>(p);
    else
        long_intervals_kernel<DW_SIGNAL_LINEAR><<<long_grid, 256, 0, stream>>>(p);
    count_launch();

    if (wj) {
        if (wj->nb > 0) {
            const unsigned g = (unsigned)std::min<int64_t>(num_sms() * 4, ceil_div(wj->nb * 32, 256));
            if (sig->kind == DW_SIGNAL_STEP)
                window_partials_kernel<DW_SIGNAL_STEP><<<g, 256, 0, stream>>>(p, wj->wp, wj->blo, wj->bhi, wj->nb,
                                                                              wj->part);
            else
                window_partials_kernel<DW_SIGNAL_LINEAR><<<g, 256, 0, stream>>>(p, wj->wp, wj->blo, wj->bhi,
                                                                                wj->nb, wj->part);
            count_launch();
        }
        tile_range_kernel<<<1, 32, 0, stream>>>(p, wj->t0, wj->t1, wj->tile_fx);
        count_launch();
    }
    if (ledger) {
        double *op_total = nullptr;
        if (ops_for_total && ops_for_total->n > 0) {
            op_total = (double *)(base + L.sum_out);
            unsigned blocks = sum_grid(ops_for_total->n);
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

int dw_attribute_window(const dw_signal_t *sig, dw_interval_set_t *sets, int32_t nsets, const dw_window_t *win,
                        const int64_t *d_blo, const int64_t *d_bhi, int64_t nb, int64_t *d_part,
                        int64_t *d_tile_fx, void *d_workspace, size_t workspace_bytes, dw_stream_t stream) {
    if (!win || (nb && (!d_blo || !d_bhi || !d_part)) || !d_tile_fx || nb < 0) return DW_E_ARG;
    if (win->g_off % TILE) return DW_E_ARG;  // the local tile grid must be the global one
    WindowJob wj{};
    wj.wp = WindowParams{win->g_off, win->n_samples_global, win->piece_lo, win->piece_hi,
                         win->ts_first, win->ts_last, win->w_first, win->w_last};
    wj.blo = d_blo;
    wj.bhi = d_bhi;
    wj.nb = nb;
    wj.part = (unsigned long long *)d_part;
    const int64_t ntl = ceil_div(sig->n, TILE);
    wj.t0 = std::min<int64_t>(std::max<int64_t>((win->piece_lo - win->g_off) / TILE, 0), ntl);
    wj.t1 = std::min<int64_t>(std::max<int64_t>(ceil_div(win->piece_hi - win->g_off, TILE), wj.t0), ntl);
    wj.tile_fx = (unsigned long long *)d_tile_fx;
    return attribute_impl(sig, sets, nsets, d_workspace, workspace_bytes, (cudaStream_t)stream, false, nullptr,
                          &wj);
}

int dw_set_attribute_sms(int n) {
    if (n < 0) return DW_E_ARG;
    g_attr_sms = n;
    return DW_OK;
}

int dw_fx_sum_exact(const double *d_x, int64_t n, int64_t *d_out_fx, void *d_workspace, size_t ws_bytes,
                    dw_stream_t stream) {
    if (n < 0 || !d_out_fx || !d_workspace || ws_bytes < dw_fx_sum_workspace_size(n)) return DW_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    if (n == 0) {
        cudaMemsetAsync(d_out_fx, 0, 16, s);
        DW_CHECK_LAUNCH();
        return DW_OK;
    }
    char *base = (char *)d_workspace;
    unsigned blocks = sum_grid(n);
    unsigned int *done = (unsigned int *)(base + 16 * (size_t)SUM_BLOCKS);
    cudaMemsetAsync(done, 0, 16, s);
    fx_sum_kernel<<<blocks, SUM_THREADS, 0, s>>>(d_x, n, (unsigned long long *)base, done, nullptr,
                                                 (unsigned long long *)d_out_fx);
    count_launch();
    DW_CHECK_LAUNCH();
    return DW_OK;
}

static_assert(STATUS_BYTES == DW_STATUS_BYTES, "status block size");

int dw_status_copy(const void *d_workspace, void *h_block, dw_stream_t stream) {
    if (!d_workspace || !h_block) return DW_E_ARG;
    return cudaMemcpyAsync(h_block, d_workspace, sizeof(DevStatus), cudaMemcpyDeviceToHost,
                           (cudaStream_t)stream) == cudaSuccess ? DW_OK : DW_E_CUDA;
}

int dw_status(const void *d_workspace, dw_stream_t stream, dw_status_t *out) {
    if (!d_workspace || !out) return DW_E_ARG;
    DevStatus st;
    if (dw_status_copy(d_workspace, &st, stream) != DW_OK) return DW_E_CUDA;
    if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return DW_E_CUDA;
    return dw_status_decode(&st, out);
}

int dw_status_decode(const void *h_block, dw_status_t *out) {
    if (!h_block || !out) return DW_E_ARG;
    DevStatus st;
    memcpy(&st, h_block, sizeof(st));
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
    unsigned blocks = sum_grid(n);
    unsigned int *done = (unsigned int *)(base + 16 * (size_t)SUM_BLOCKS);
    cudaMemsetAsync(done, 0, 16, s);
    fx_sum_kernel<<<blocks, SUM_THREADS, 0, s>>>(d_x, n, (unsigned long long *)base, done, d_out);
    count_launch();
    DW_CHECK_LAUNCH();
    return DW_OK;
}

#ifdef DW_PHASE_PROF
int dw_phase_prof(unsigned long long *out16, int reset) {
    if (cudaMemcpyFromSymbol(out16, g_phase, sizeof(g_phase)) != cudaSuccess) return DW_E_CUDA;
    if (reset) {
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(g_phase, z, sizeof(z));
    }
    return DW_OK;
}
#endif

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
