/*
 * dw_oracle.c -- CPU restatement of the reference's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker for the CUDA path, and the
 * CPU baseline that bench.py times; the product (paper_2512_08365_b200/) never
 * links or calls it.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs load it.
 *
 * Parity is PINNED: tests/test_oracle.py checks every function below against
 * the golden vectors that tests/golden/make_golden.py recorded by running the
 * reference package itself (/root/reference/pkg/src/diffwatt).
 *
 * What each function restates (reference = /root/reference/pkg/src/diffwatt):
 *
 *   dwo_integrate_step    energy.integrate, ground-truth branch (energy.py:90-104)
 *                         over PowerSignal.from_breakpoints segments (energy.py:68-82).
 *                         The reference loops over EVERY segment and adds w*overlap
 *                         only when overlap > 0; we binary-search the first
 *                         overlapping segment and add exactly the same terms in the
 *                         same order, so the result is bit-identical (no FMA:
 *                         compile with -ffp-contract=off).
 *   dwo_integrate_linear  energy._integrate_samples (energy.py:108-130): trapezoid over
 *                         [lo] + {ts in (lo,hi)} + [hi] with value() taking the FIRST
 *                         bracketing sample pair (energy.py:115-124).
 *   dwo_*_fx              the same terms, accumulated exactly in 2^-32 W*us fixed
 *                         point (int128) and rounded once: the definition the GPU
 *                         uses for intervals longer than DW_DIRECT_MAX segments
 *                         (DESIGN.md "long intervals").  Not in the reference; it is
 *                         pinned to the reference through dwo_integrate_* (tests
 *                         bound the difference at 1e-12 relative).
 *   dwo_detect            detect.detect_waste per-pair rule (detect.py:90-126) and
 *                         _segment_latency (detect.py:48-52), given per-pair output
 *                         diffs (the tensor part, detect.py:55-69, is host-side).
 *   dwo_rank              detect.report ordering (detect.py:263-266): key
 *                         (verdict != waste, -wasted_joules, nodes_a) with a stable
 *                         sort; nodes_a order is passed in as an integer tie rank.
 *   dwo_join              the signature join (DESIGN.md "signature
 *                         join"): (sig, k-th occurrence in op order).  Parity
 *                         unpinned against the reference (it has no such join), so
 *                         this restates OUR written definition.
 *
 * Build: see oracle/Makefile (gcc -O2 -pthread -ffp-contract=off -shared -fPIC).
 * Per-interval work is spread over host threads (pthreads; the image's gcc has
 * no libgomp); each interval's sum is sequential, so results do not depend on
 * the thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#include <pthread.h>
#include <unistd.h>

#define US_PER_S 1000000.0

/* errors (same numbering as include/dwb200.h) */
#define DW_OK 0
#define DW_E_REVERSED (-1) /* "interval end precedes start" */
#define DW_E_SPAN (-2)     /* "interval [lo,hi] outside signal span [s,e]" */
#define DW_E_EMPTY (-3)    /* "empty power signal" */
#define DW_E_ARG (-5)

#define DW_DIRECT_MAX 256 /* see include/dwb200.h */
#define DW_TILE 1024
#define DW_TILE_THREADS 192

typedef __int128 i128;

/* ---------------------------------------------------------------- threads */

static int g_threads = 0; /* 0 = all online cores */

void dwo_set_threads(int n) { g_threads = n; }

int dwo_num_threads(void) {
    if (g_threads > 0) return g_threads;
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

typedef void (*range_fn)(void *ctx, int64_t lo, int64_t hi);
typedef struct { range_fn fn; void *ctx; int64_t lo, hi; } par_job;

static void *par_thread(void *p) {
    par_job *j = (par_job *)p;
    j->fn(j->ctx, j->lo, j->hi);
    return NULL;
}

static void par_for(int64_t n, range_fn fn, void *ctx) {
    int nt = dwo_num_threads();
    if (nt > 64) nt = 64;
    if (n < 4096 || nt == 1) { fn(ctx, 0, n); return; }
    pthread_t th[64];
    par_job jobs[64];
    int ok[64];
    int64_t chunk = (n + nt - 1) / nt;
    for (int t = 0; t < nt; t++) {
        jobs[t].fn = fn;
        jobs[t].ctx = ctx;
        jobs[t].lo = t * chunk < n ? t * chunk : n;
        jobs[t].hi = (t + 1) * chunk < n ? (t + 1) * chunk : n;
        ok[t] = pthread_create(&th[t], NULL, par_thread, &jobs[t]) == 0;
        if (!ok[t]) fn(ctx, jobs[t].lo, jobs[t].hi);
    }
    for (int t = 0; t < nt; t++)
        if (ok[t]) pthread_join(th[t], NULL);
}

/* ---------------------------------------------------------------- helpers */

/* first index i in [0,n) with a[i] >= key (n if none) */
static int64_t lower_bound64(const int64_t *a, int64_t n, int64_t key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = lo + ((hi - lo) >> 1);
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* first index i with a[i] > key */
static int64_t upper_bound64(const int64_t *a, int64_t n, int64_t key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = lo + ((hi - lo) >> 1);
        if (a[mid] <= key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* Fixed point: q_s(x) = round-half-even(x * 2^s) as int128.
 *   s = DW_FX_TERM_BITS (40) for integrand terms in W*us,
 *   s = DW_FX_JOULE_BITS (64) for sums of joules. */
#define DW_FX_TERM_BITS 40
#define DW_FX_JOULE_BITS 64

static i128 fx_from_double(double x, int scale) {
    if (x == 0.0) return 0;
    uint64_t bits;
    memcpy(&bits, &x, 8);
    int neg = (int)(bits >> 63);
    int e = (int)((bits >> 52) & 0x7ff);
    uint64_t m = bits & 0xfffffffffffffULL;
    if (e == 0) e = 1; else m |= 1ULL << 52;
    /* x = m * 2^(e-1075);  x*2^scale = m * 2^(e-1075+scale) */
    int sh = e - 1075 + scale;
    i128 v;
    if (sh >= 0) {
        v = (i128)m << sh;
    } else {
        int r = -sh;
        if (r >= 64) {
            v = 0; /* m < 2^53 -> m*2^-64 < 0.5 */
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

/* round-half-even int128 -> double, then * 2^-scale */
static double fx_to_double(i128 v, int scale) {
    int neg = v < 0;
    unsigned __int128 u = neg ? (unsigned __int128)(-v) : (unsigned __int128)v;
    double r;
    if ((u >> 53) == 0) {
        r = (double)(uint64_t)u;
    } else {
        int len = 128;
        uint64_t hi = (uint64_t)(u >> 64), lo = (uint64_t)u;
        len = hi ? 128 - __builtin_clzll(hi) : 64 - __builtin_clzll(lo);
        int drop = len - 53;
        unsigned __int128 q = u >> drop;
        unsigned __int128 rem = u & ((((unsigned __int128)1) << drop) - 1);
        unsigned __int128 half = ((unsigned __int128)1) << (drop - 1);
        if (rem > half || (rem == half && (q & 1))) q++;
        r = ldexp((double)(uint64_t)q, drop); /* q <= 2^53: exact */
    }
    r = ldexp(r, -scale);
    return neg ? -r : r;
}

#define q_term(x) fx_from_double((x), DW_FX_TERM_BITS)
#define term_to_joules(v) (fx_to_double((v), DW_FX_TERM_BITS) / US_PER_S)

/* -------------------------------------------------------- step (ground truth) */

/* segment i: [ts[i], ts[i+1]) for i < n-1; last: [ts[n-1], span_hi) */
static inline int64_t seg_end(const int64_t *ts, int64_t n, int64_t span_hi, int64_t i) {
    return i + 1 < n ? ts[i + 1] : span_hi;
}

static int check_iv(int64_t lo, int64_t hi, int64_t span_lo, int64_t span_hi) {
    if (hi < lo) return DW_E_REVERSED;
    if (lo < span_lo || hi > span_hi) return DW_E_SPAN;
    return DW_OK;
}

/* number of segments the interval overlaps with positive length */
static int64_t step_nseg(const int64_t *ts, int64_t n, int64_t lo, int64_t hi) {
    if (hi <= lo) return 0;
    int64_t a = upper_bound64(ts, n, lo) - 1;      /* last ts <= lo */
    int64_t b = lower_bound64(ts, n, hi) - 1;      /* last ts < hi  */
    return b - a + 1;
}

static double step_direct(const int64_t *ts, const double *w, int64_t n, int64_t span_hi,
                          int64_t lo, int64_t hi) {
    double total = 0.0;
    if (hi > lo) {
        int64_t i = upper_bound64(ts, n, lo) - 1;
        if (i < 0) i = 0;
        for (; i < n && ts[i] < hi; i++) {
            int64_t s = ts[i], e = seg_end(ts, n, span_hi, i);
            int64_t ov = (e < hi ? e : hi) - (s > lo ? s : lo);
            if (ov > 0) total += w[i] * (double)ov;
        }
    }
    return total / US_PER_S;
}

/* ---- the device's fixed-point definition (MODE_DEVICE long intervals,
 * MODE_EXACT every interval) ----
 * The interval's pieces (the reference's own decomposition: edge pieces with
 * the interpolated endpoint values, interior pieces between samples) are each
 * rounded to 2^-40 W*us and summed exactly (int128); the sum is rounded once
 * to a double and divided by 1e6.  Integer addition is associative, so the
 * GPU may group the pieces any way it likes (window prefixes, whole-tile
 * sums) and still return exactly this value. */
typedef double (*term_fn)(const void *ctx, int64_t i);

/* exact sum of terms [j0, j1] */
static i128 fx_range(term_fn term, const void *ctx, int64_t nterms, int64_t j0, int64_t j1) {
    (void)nterms;
    i128 acc = 0;
    for (int64_t i = j0; i <= j1; i++) acc += q_term(term(ctx, i));
    return acc;
}

typedef struct { const int64_t *ts; const double *w; int64_t n, span_hi; } sig_ctx;

static double step_term(const void *c, int64_t i) {
    const sig_ctx *s = (const sig_ctx *)c;
    return s->w[i] * (double)(seg_end(s->ts, s->n, s->span_hi, i) - s->ts[i]);
}

static double step_fx(const int64_t *ts, const double *w, int64_t n, int64_t span_hi,
                      int64_t lo, int64_t hi) {
    sig_ctx c = {ts, w, n, span_hi};
    int64_t a = upper_bound64(ts, n, lo) - 1;
    int64_t b = lower_bound64(ts, n, hi) - 1;
    i128 acc = fx_range(step_term, &c, n, a + 1, b - 1);
    acc += q_term(w[a] * (double)(ts[a + 1] - lo));
    int64_t eb = seg_end(ts, n, span_hi, b);
    acc += q_term(w[b] * (double)((eb < hi ? eb : hi) - ts[b]));
    return term_to_joules(acc);
}

/* MODE_EXACT, step: every interval as the exact sum of its pieces.  Pieces
 * as the device's exact path takes them: none for hi == lo; one
 * w[a]*(hi-lo) inside a single segment; else the first partial segment, the
 * whole interior segments and the last partial segment. */
static double step_exact(const int64_t *ts, const double *w, int64_t n, int64_t span_hi,
                         int64_t lo, int64_t hi) {
    if (hi <= lo) return 0.0;
    sig_ctx c = {ts, w, n, span_hi};
    int64_t a = upper_bound64(ts, n, lo) - 1;
    int64_t b = lower_bound64(ts, n, hi) - 1;
    if (a == b) return term_to_joules(q_term(w[a] * (double)(hi - lo)));
    i128 acc = fx_range(step_term, &c, n, a + 1, b - 1);
    acc += q_term(w[a] * (double)(ts[a + 1] - lo));
    acc += q_term(w[b] * (double)(hi - ts[b]));
    return term_to_joules(acc);
}

/* the ledger total over the whole span, device definition */
double dwo_total_device(int kind, const int64_t *ts, const double *w, int64_t n, int64_t span_hi);

typedef struct {
    const int64_t *ts; const double *w; int64_t n, span_hi;
    const int64_t *lo, *hi; double *out; int mode;
} iv_job;

static void step_range(void *ctx, int64_t k0, int64_t k1) {
    iv_job *j = (iv_job *)ctx;
    for (int64_t k = k0; k < k1; k++) {
        if (j->mode == 2)
            j->out[k] = step_exact(j->ts, j->w, j->n, j->span_hi, j->lo[k], j->hi[k]);
        else if (j->mode == 1 && step_nseg(j->ts, j->n, j->lo[k], j->hi[k]) > DW_DIRECT_MAX)
            j->out[k] = step_fx(j->ts, j->w, j->n, j->span_hi, j->lo[k], j->hi[k]);
        else
            j->out[k] = step_direct(j->ts, j->w, j->n, j->span_hi, j->lo[k], j->hi[k]);
    }
}

/* mode: 0 = reference-literal sequential sum for every interval;
 *       1 = the GPU's reference-order mode: sequential for <= DW_DIRECT_MAX
 *           segments, exact fixed point above;
 *       2 = the GPU's exact mode (DW_SUM_EXACT): exact fixed point for every
 *           interval.
 * Returns DW_OK, or the error code of the first bad interval (*bad = index). */
int dwo_integrate_step(const int64_t *ts, const double *w, int64_t n, int64_t span_hi,
                       const int64_t *lo, const int64_t *hi, int64_t m, double *out,
                       int mode, int64_t *bad) {
    if (n <= 0) { if (bad) *bad = -1; return DW_E_EMPTY; }
    int64_t span_lo = ts[0];
    for (int64_t k = 0; k < m; k++) {
        int rc = check_iv(lo[k], hi[k], span_lo, span_hi);
        if (rc) { if (bad) *bad = k; return rc; }
    }
    iv_job j = {ts, w, n, span_hi, lo, hi, out, mode};
    par_for(m, step_range, &j);
    return DW_OK;
}

/* ------------------------------------------------------ linear (trapezoid) */

/* value(t) of energy.py:115-124 at an integer time t */
static double lin_value(const int64_t *ts, const double *w, int64_t n, int64_t t) {
    if (t <= ts[0]) return w[0];
    if (t >= ts[n - 1]) return w[n - 1];
    int64_t i = lower_bound64(ts, n, t) - 1; /* first i with ts[i] <= t <= ts[i+1] */
    double frac = (double)(t - ts[i]) / (double)(ts[i + 1] - ts[i]);
    return w[i] + frac * (w[i + 1] - w[i]);
}

static inline double lin_term(const int64_t *ts, const double *w, int64_t n, int64_t a,
                              int64_t b) {
    return 0.5 * (lin_value(ts, w, n, a) + lin_value(ts, w, n, b)) * (double)(b - a);
}

/* pieces of the trapezoid = 1 + #{ts in (lo, hi)} */
static int64_t lin_npieces(const int64_t *ts, int64_t n, int64_t lo, int64_t hi) {
    int64_t first = upper_bound64(ts, n, lo);
    int64_t last = lower_bound64(ts, n, hi);
    int64_t interior = last > first ? last - first : 0;
    return interior + 1;
}

static double lin_sample(const int64_t *ts, const double *w, int64_t n, int64_t j) {
    (void)ts;
    if (j == 0) return w[0];
    if (j == n - 1) return w[n - 1];
    return w[j - 1] + 1.0 * (w[j] - w[j - 1]);
}

static double lin_piece_term(const void *c, int64_t j) {
    const sig_ctx *s = (const sig_ctx *)c;
    return 0.5 * (lin_sample(s->ts, s->w, s->n, j) + lin_sample(s->ts, s->w, s->n, j + 1)) *
           (double)(s->ts[j + 1] - s->ts[j]);
}

static double lin_fx(const int64_t *ts, const double *w, int64_t n, int64_t lo, int64_t hi) {
    sig_ctx c = {ts, w, n, 0};
    int64_t first = upper_bound64(ts, n, lo);
    int64_t last = lower_bound64(ts, n, hi);
    i128 acc = fx_range(lin_piece_term, &c, n - 1, first, last - 2);
    acc += q_term(lin_term(ts, w, n, lo, ts[first]));
    acc += q_term(lin_term(ts, w, n, ts[last - 1], hi));
    return term_to_joules(acc);
}

static double lin_integrate(const int64_t *ts, const double *w, int64_t n, int64_t lo,
                            int64_t hi, int fx) {
    if (fx) {
        /* one piece [lo, hi] when no sample lies strictly inside */
        if (lin_npieces(ts, n, lo, hi) == 1) return term_to_joules(q_term(lin_term(ts, w, n, lo, hi)));
        return lin_fx(ts, w, n, lo, hi);
    }
    int64_t first = upper_bound64(ts, n, lo); /* first ts > lo */
    int64_t last = lower_bound64(ts, n, hi);  /* first ts >= hi */
    int64_t prev = lo;
    double total = 0.0;
    i128 acc = 0;
    for (int64_t j = first; j < last; j++) {
        double t = lin_term(ts, w, n, prev, ts[j]);
        if (fx) acc += q_term(t); else total += t;
        prev = ts[j];
    }
    double t = lin_term(ts, w, n, prev, hi);
    if (fx) { acc += q_term(t); return term_to_joules(acc); }
    total += t;
    return total / US_PER_S;
}

static void lin_range(void *ctx, int64_t k0, int64_t k1) {
    iv_job *j = (iv_job *)ctx;
    for (int64_t k = k0; k < k1; k++) {
        int fx = j->mode == 2 || (j->mode == 1 && lin_npieces(j->ts, j->n, j->lo[k], j->hi[k]) > DW_DIRECT_MAX);
        j->out[k] = lin_integrate(j->ts, j->w, j->n, j->lo[k], j->hi[k], fx);
    }
}

int dwo_integrate_linear(const int64_t *ts, const double *w, int64_t n, const int64_t *lo,
                         const int64_t *hi, int64_t m, double *out, int mode, int64_t *bad) {
    if (n <= 0) { if (bad) *bad = -1; return DW_E_EMPTY; }
    for (int64_t k = 0; k < m; k++) {
        int rc = check_iv(lo[k], hi[k], ts[0], ts[n - 1]);
        if (rc) { if (bad) *bad = k; return rc; }
    }
    iv_job j = {ts, w, n, 0, lo, hi, out, mode};
    par_for(m, lin_range, &j);
    return DW_OK;
}

/* Exact fixed-point (2^-64 J) sum of joule values, rounded once: the GPU's
 * definition of large reductions (operator_total, report wasted_joules). */
double dwo_fx_sum(const double *x, int64_t n) {
    i128 acc = 0;
    for (int64_t i = 0; i < n; i++) acc += fx_from_double(x[i], DW_FX_JOULE_BITS);
    return fx_to_double(acc, DW_FX_JOULE_BITS);
}

/* CPython >= 3.12 builtin sum() over floats (Neumaier compensation; the
 * reference's operator_total energy.py:274, subgraph_joules energy.py:277 and
 * report's wasted_joules detect.py:267 all go through it). */
typedef struct { double f, c; int64_t n; } py_sum_t;

static inline void py_sum_add(py_sum_t *s, double x) {
    if (s->n++ == 0) { s->f = x; s->c = 0.0; return; }
    double t = s->f + x;
    if (fabs(s->f) >= fabs(x)) s->c += (s->f - t) + x;
    else s->c += (x - t) + s->f;
    s->f = t;
}

static inline double py_sum_result(const py_sum_t *s) {
    if (s->n == 0) return 0.0;
    double f = s->f;
    if (s->c != 0.0 && isfinite(s->c)) f += s->c;
    return f;
}

double dwo_py_sum(const double *x, int64_t n) {
    py_sum_t s = {0.0, 0.0, 0};
    for (int64_t i = 0; i < n; i++) py_sum_add(&s, x[i]);
    return py_sum_result(&s);
}

/* ------------------------------------------------------------------ detect */

#define V_BELOW 0
#define V_TRADEOFF 1
#define V_WASTE 2
#define SIDE_NONE 0
#define SIDE_A 1
#define SIDE_B 2

/* Per pair: members are CSR over op indices of each side.  Outputs per pair:
 * energy[2], ratio, lat[2], verdict, side, wasted, informational. */
int dwo_detect(int64_t P, const int64_t *off_a, const int32_t *mem_a, const int64_t *off_b,
               const int32_t *mem_b, const double *joules_a, const double *joules_b,
               const int64_t *start_a, const int64_t *end_a, const int64_t *start_b,
               const int64_t *end_b, const double *out_diff, double threshold,
               double *energy, double *ratio, int64_t *lat, int8_t *verdict, int8_t *side,
               double *wasted, int8_t *informational) {
    if (!(threshold > 0.0 && threshold <= 1.0)) return DW_E_ARG;
    for (int64_t p = 0; p < P; p++) {
        py_sum_t sa = {0.0, 0.0, 0}, sb = {0.0, 0.0, 0};
        int64_t smin = 0, emax = 0;
        for (int64_t k = off_a[p]; k < off_a[p + 1]; k++) {
            int32_t o = mem_a[k];
            py_sum_add(&sa, joules_a[o]);
            if (k == off_a[p] || start_a[o] < smin) smin = start_a[o];
            if (k == off_a[p] || end_a[o] > emax) emax = end_a[o];
        }
        int64_t la = off_a[p + 1] > off_a[p] ? emax - smin : 0;
        for (int64_t k = off_b[p]; k < off_b[p + 1]; k++) {
            int32_t o = mem_b[k];
            py_sum_add(&sb, joules_b[o]);
            if (k == off_b[p] || start_b[o] < smin) smin = start_b[o];
            if (k == off_b[p] || end_b[o] > emax) emax = end_b[o];
        }
        int64_t lb = off_b[p + 1] > off_b[p] ? emax - smin : 0;
        double ea = py_sum_result(&sa), eb = py_sum_result(&sb);
        double high = ea >= eb ? ea : eb, low = ea >= eb ? eb : ea;
        double r;
        int sd;
        if (high == low) { r = 1.0; sd = SIDE_NONE; }
        else { r = low > 0 ? high / low : INFINITY; sd = ea > eb ? SIDE_A : SIDE_B; }
        int v;
        if (r >= 1.0 + threshold) {
            int64_t eff = sd == SIDE_A ? lb : la, ineff = sd == SIDE_A ? la : lb;
            double od = out_diff ? out_diff[p] : 0.0;
            v = ((double)eff <= 1.01 * (double)ineff && od <= 0.01) ? V_WASTE : V_TRADEOFF;
        } else {
            v = V_BELOW;
        }
        energy[2 * p] = ea;
        energy[2 * p + 1] = eb;
        ratio[p] = r;
        lat[2 * p] = la;
        lat[2 * p + 1] = lb;
        verdict[p] = (int8_t)v;
        side[p] = (int8_t)sd;
        wasted[p] = high - low;
        informational[p] = (int8_t)(v == V_BELOW && r >= 1.0 + 0.05);
    }
    return DW_OK;
}

/* ------------------------------------------------------------------- rank */

typedef struct { int waste; double wasted; int64_t tie; int64_t idx; } rank_rec;

static int rank_cmp(const void *pa, const void *pb) {
    const rank_rec *a = (const rank_rec *)pa, *b = (const rank_rec *)pb;
    if (a->waste != b->waste) return a->waste ? -1 : 1;
    if (a->wasted != b->wasted) return a->wasted > b->wasted ? -1 : 1;
    if (a->tie != b->tie) return a->tie < b->tie ? -1 : 1;
    return a->idx < b->idx ? -1 : (a->idx > b->idx); /* stable */
}

/* order[r] = index of the finding ranked r.  tie[i] = rank of nodes_a under
 * Python tuple ordering (equal tuples share a rank). */
int dwo_rank(int64_t P, const int8_t *verdict, const double *wasted, const int64_t *tie,
             int64_t *order) {
    rank_rec *r = (rank_rec *)malloc(sizeof(rank_rec) * (P > 0 ? P : 1));
    if (!r) return DW_E_ARG;
    for (int64_t i = 0; i < P; i++) {
        r[i].waste = verdict[i] == V_WASTE;
        r[i].wasted = wasted[i];
        r[i].tie = tie[i];
        r[i].idx = i;
    }
    qsort(r, (size_t)P, sizeof(rank_rec), rank_cmp);
    for (int64_t i = 0; i < P; i++) order[i] = r[i].idx;
    free(r);
    return DW_OK;
}

/* ------------------------------------------------------------------- join */

typedef struct { uint64_t sig; int64_t idx; } sig_rec;

static int sig_cmp(const void *pa, const void *pb) {
    const sig_rec *a = (const sig_rec *)pa, *b = (const sig_rec *)pb;
    if (a->sig != b->sig) return a->sig < b->sig ? -1 : 1;
    return a->idx < b->idx ? -1 : (a->idx > b->idx);
}

/* occ[i] = #{j < i : sig[j] == sig[i]} (ops are in time order by index) */
int dwo_occurrence(const uint64_t *sig, int64_t n, int64_t *occ) {
    sig_rec *r = (sig_rec *)malloc(sizeof(sig_rec) * (n > 0 ? n : 1));
    if (!r) return DW_E_ARG;
    for (int64_t i = 0; i < n; i++) { r[i].sig = sig[i]; r[i].idx = i; }
    qsort(r, (size_t)n, sizeof(sig_rec), sig_cmp);
    for (int64_t i = 0; i < n; i++)
        occ[r[i].idx] = (i > 0 && r[i - 1].sig == r[i].sig) ? occ[r[i - 1].idx] + 1 : 0;
    free(r);
    return DW_OK;
}

/* match_a[i] = B index with equal (sig, occ) or -1; match_b likewise. */
int dwo_join(const uint64_t *sig_a, int64_t na, const uint64_t *sig_b, int64_t nb,
             int64_t *match_a, int64_t *match_b) {
    int64_t *occ_a = (int64_t *)malloc(sizeof(int64_t) * (na > 0 ? na : 1));
    int64_t *occ_b = (int64_t *)malloc(sizeof(int64_t) * (nb > 0 ? nb : 1));
    sig_rec *rb = (sig_rec *)malloc(sizeof(sig_rec) * (nb > 0 ? nb : 1));
    if (!occ_a || !occ_b || !rb) return DW_E_ARG;
    dwo_occurrence(sig_a, na, occ_a);
    dwo_occurrence(sig_b, nb, occ_b);
    for (int64_t j = 0; j < nb; j++) { rb[j].sig = sig_b[j]; rb[j].idx = j; match_b[j] = -1; }
    qsort(rb, (size_t)nb, sizeof(sig_rec), sig_cmp); /* (sig, idx) == (sig, occ) order */
    for (int64_t i = 0; i < na; i++) {
        match_a[i] = -1;
        /* first B record with this sig, then step occ_a[i] */
        int64_t lo = 0, hi = nb;
        while (lo < hi) {
            int64_t mid = lo + ((hi - lo) >> 1);
            if (rb[mid].sig < sig_a[i]) lo = mid + 1; else hi = mid;
        }
        int64_t k = lo + occ_a[i];
        if (k < nb && rb[k].sig == sig_a[i]) {
            match_a[i] = rb[k].idx;
            match_b[rb[k].idx] = i;
        }
    }
    free(occ_a);
    free(occ_b);
    free(rb);
    return DW_OK;
}


/* exact: 1 = DW_SUM_EXACT (every span as the exact sum of its pieces); 0 =
 * reference order (the literal sequential sum up to DW_DIRECT_MAX pieces). */
double dwo_total_device_mode(int kind, const int64_t *ts, const double *w, int64_t n, int64_t span_hi,
                             int exact) {
    sig_ctx c = {ts, w, n, span_hi};
    int64_t nterms = kind == 0 ? n : (n > 1 ? n - 1 : 1);
    if (nterms <= DW_DIRECT_MAX && !exact) {
        int64_t lo = ts[0], hi = kind == 0 ? span_hi : ts[n - 1];
        if (kind == 0) return step_direct(ts, w, n, span_hi, lo, hi);
        return lin_integrate(ts, w, n, lo, hi, 0);
    }
    if (kind != 0 && n == 1) return 0.0;
    return term_to_joules(fx_range(kind == 0 ? step_term : lin_piece_term, &c, nterms, 0, nterms - 1));
}

double dwo_total_device(int kind, const int64_t *ts, const double *w, int64_t n, int64_t span_hi) {
    return dwo_total_device_mode(kind, ts, w, n, span_hi, 0);
}

/* ---------------------------------------------------- overlap split (G1)
 * The builder's definition (no reference function
 * exists -- SURVEY.md G1).  Within one interval set, at every instant the
 * signal's power is divided equally among the intervals active then:
 *   x_0 < ... < x_u-1  the distinct endpoints of the set's non-empty intervals
 *   slice k = [x_k, x_k+1], c_k = intervals with start <= x_k and end >= x_k+1
 *   e_k = the compat integral of slice k (MODE_DEVICE: bit-identical to the
 *         reference's sequential sum up to DW_DIRECT_MAX segments)
 *   share_k = e_k / c_k (IEEE), 0 when c_k == 0
 *   joules(i) = share_k when interval i is the single slice k, otherwise the
 *               exact (2^-64 J fixed point) sum of its slices' shares, rounded
 *               once; 0 for an empty interval.
 * With no overlap every interval is one slice with c = 1, so split == compat
 * exactly.  kind: 0 step, 1 linear. */
typedef struct { int64_t t; int32_t d; } split_ev;

static int split_ev_cmp(const void *pa, const void *pb) {
    int64_t a = ((const split_ev *)pa)->t, b = ((const split_ev *)pb)->t;
    return a < b ? -1 : a > b;
}

int dwo_split(int kind, const int64_t *ts, const double *w, int64_t n, int64_t span_hi,
              const int64_t *lo, const int64_t *hi, int64_t m, double *out, int64_t *bad) {
    if (n <= 0) { if (bad) *bad = -1; return DW_E_EMPTY; }
    int64_t span_end = kind == 0 ? span_hi : ts[n - 1];
    for (int64_t k = 0; k < m; k++) {
        int rc = check_iv(lo[k], hi[k], ts[0], span_end);
        if (rc) { if (bad) *bad = k; return rc; }
    }
    split_ev *ev = (split_ev *)malloc(sizeof(split_ev) * (size_t)(2 * m + 1));
    int64_t ne = 0;
    for (int64_t k = 0; k < m; k++) {
        if (hi[k] == lo[k]) continue;
        ev[ne].t = lo[k]; ev[ne++].d = 1;
        ev[ne].t = hi[k]; ev[ne++].d = -1;
    }
    qsort(ev, (size_t)ne, sizeof(split_ev), split_ev_cmp);
    int64_t *x = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ne + 1));
    int64_t *c = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ne + 1));
    int64_t u = 0, run = 0;
    for (int64_t e = 0; e < ne; e++) {
        run += ev[e].d;
        if (e + 1 == ne || ev[e + 1].t != ev[e].t) { x[u] = ev[e].t; c[u] = run; u++; }
    }
    int64_t ns = u > 1 ? u - 1 : 0;
    double *es = (double *)malloc(sizeof(double) * (size_t)(ns + 1));
    i128 *P = (i128 *)malloc(sizeof(i128) * (size_t)(u + 1));
    int rc = DW_OK;
    if (ns) {
        rc = kind == 0 ? dwo_integrate_step(ts, w, n, span_hi, x, x + 1, ns, es, 1, bad)
                       : dwo_integrate_linear(ts, w, n, x, x + 1, ns, es, 1, bad);
    }
    if (rc == DW_OK) {
        P[0] = 0;
        for (int64_t k = 0; k < ns; k++) {
            es[k] = c[k] > 0 ? es[k] / (double)c[k] : 0.0;
            P[k + 1] = P[k] + fx_from_double(es[k], DW_FX_JOULE_BITS);
        }
        for (int64_t k = 0; k < m; k++) {
            if (hi[k] == lo[k]) { out[k] = 0.0; continue; }
            int64_t a = lower_bound64(x, u, lo[k]), b = lower_bound64(x, u, hi[k]);
            out[k] = b == a + 1 ? es[a] : fx_to_double(P[b] - P[a], DW_FX_JOULE_BITS);
        }
    }
    free(ev); free(x); free(c); free(es); free(P);
    return rc;
}

/* ------------------------------------------------------- replay estimator
 * replay_estimate (energy.py:196-256) for every operator, restated: the op's
 * truth profile tiled `repeat` times, read by the delayed sampler
 * (energy.py:144-171; the delays are the numpy stream, drawn by the caller:
 * every op restarts the same seeded stream, so one array serves all ops),
 * mid-window samples averaged with Python's sum().  Truth: breakpoints
 * ts/w with the last segment ending at span_hi.  Returns DW_OK or
 * DW_E_EMPTY with *bad = the first op whose profile is empty (the reference's
 * "sample_signal requires a ground-truth signal"). */
static double replay_value(const int64_t *ts, const double *w, int64_t n, int64_t span_hi, int64_t start,
                           int64_t d, int64_t repeat, int64_t i0, int64_t i1, int64_t p0s, int64_t ple,
                           double x) {
    /* tiled segments: tile k, truth segment i in [i0, i1]:
       [k d + max(ts_i, start) - start, k d + min(end_i, start + d) - start) */
    const double sr = (double)p0s, er = (double)((repeat - 1) * d + ple);
    if (x < sr) x = sr;
    if (x > er) x = er;
    int64_t k = (int64_t)(x / (double)d);
    if (k < 0) k = 0;
    if (k > repeat - 1) k = repeat - 1;
    while (k > 0 && (double)(k * d + p0s) > x) k--;
    while (k < repeat - 1 && (double)((k + 1) * d + p0s) <= x) k++;
    const int64_t base = k * d - start;
    for (int64_t i = i0; i <= i1; i++) {  /* first containing segment */
        int64_t s = ts[i] > start ? ts[i] : start;
        int64_t e = i + 1 < n ? ts[i + 1] : span_hi;
        if (e > start + d) e = start + d;
        if ((double)(base + s) <= x && x < (double)(base + e)) return w[i];
    }
    return w[i1]; /* no containing segment: the last tiled segment's watts */
}

int dwo_replay(const int64_t *ts, const double *w, int64_t n, int64_t span_hi, const int64_t *op_start,
               const int64_t *op_end, int64_t nops, int64_t repeat, int64_t period, const double *delays,
               int64_t ndelays, double *watts_out, double *joules_out, int64_t *bad) {
    for (int64_t o = 0; o < nops; o++) {
        const int64_t start = op_start[o], end = op_end[o], d = end - start;
        /* truth segments overlapping [start, end) */
        int64_t i0 = -1, i1 = -1;
        for (int64_t i = 0; i < n; i++) {
            int64_t s = ts[i], e = i + 1 < n ? ts[i + 1] : span_hi;
            int64_t lo = s > start ? s : start, hi = e < end ? e : end;
            if (hi > lo) { if (i0 < 0) i0 = i; i1 = i; }
        }
        if (i0 < 0) { if (bad) *bad = o; return DW_E_EMPTY; }
        const int64_t p0s = (ts[i0] > start ? ts[i0] : start) - start;
        int64_t ple = (i1 + 1 < n ? ts[i1 + 1] : span_hi);
        if (ple > end) ple = end;
        ple -= start;
        const int64_t sr = p0s, er = (repeat - 1) * d + ple;
        const double total = (double)(repeat * d);
        const double lo_m = 0.1 * total, hi_m = (1.0 - 0.1) * total;
        py_sum_t mid, all;
        memset(&mid, 0, sizeof(mid));
        memset(&all, 0, sizeof(all));
        int64_t nmid = 0, nall = 0, di = 0;
        for (int64_t t = sr + period; t <= er; t += period) {
            const double dl = di < ndelays ? delays[di] : 0.0;
            di++;
            const double v = replay_value(ts, w, n, span_hi, start, d, repeat, i0, i1, p0s, ple, (double)t - dl);
            py_sum_add(&all, v); nall++;
            if (lo_m <= (double)t && (double)t <= hi_m) { py_sum_add(&mid, v); nmid++; }
        }
        if (nall == 0) {  /* span shorter than one period: one read at the end */
            const double dl = ndelays ? delays[0] : 0.0;
            const double v = replay_value(ts, w, n, span_hi, start, d, repeat, i0, i1, p0s, ple, (double)er - dl);
            py_sum_add(&all, v); nall++;
            if (lo_m <= (double)er && (double)er <= hi_m) { py_sum_add(&mid, v); nmid++; }
        }
        const double wt = nmid ? py_sum_result(&mid) / (double)nmid : py_sum_result(&all) / (double)nall;
        watts_out[o] = wt;
        joules_out[o] = wt * (double)d / 1000000.0;
    }
    return DW_OK;
}
