/*
 * dwb200.h -- C ABI of libdwb200.so, the B200 (sm_100a) hot path of the
 * Magneton / diffwatt differential energy debugger.
 *
 * The reference (/root/reference/pkg/src/diffwatt) is pure Python and has no
 * FFI; its drop-in boundary is the Python API.  Each entry point
 * below replaces the inner loop of one reference function, and the Python
 * package paper_2512_08365_b200 binds them with ctypes behind the reference's
 * own names (build_ledger, integrate, detect_waste, report):
 *
 *   dw_attribute        energy.integrate per interval            energy.py:90-130
 *   dw_ledger           energy.build_ledger (ground_truth/sampled) energy.py:280-331
 *   dw_fx_sum           EnergyLedger.operator_total               energy.py:273-274
 *   dw_step_value_at    PowerSignal.value_at (the sampler's read) energy.py:57-66
 *   dw_detect_pairs     detect.detect_waste per-pair rule         detect.py:72-130
 *   dw_rank             detect.report ordering                    detect.py:256-278
 *   dw_rank_segmented   report ordering of every pair of a corpus    detect.py:256-278
 *   dw_join_diff        signature hash-join + deltas + verdicts   (new)
 *
 * Conventions
 *   - Every pointer argument named d_* is DEVICE memory owned by the caller.
 *     The library allocates nothing: scratch comes from a caller workspace whose
 *     size the matching *_workspace_size() returns.  Device pointers must be
 *     16-byte aligned (torch / cudaMalloc allocations are).
 *   - Calls are asynchronous on the given stream.  Data-dependent errors (an
 *     interval outside the signal, unsorted input, ...) are written into the
 *     workspace's status block; dw_status() synchronises the stream and reads it.
 *     Argument errors are returned immediately.
 *   - No global state: concurrent calls on different streams with different
 *     workspaces are safe.
 *   - Times are int64 microseconds, power fp64 watts, energy fp64 joules.
 */
#ifndef DWB200_H
#define DWB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *dw_stream_t; /* == cudaStream_t */

/* ------------------------------------------------------------- error codes */
#define DW_OK 0
#define DW_E_REVERSED (-1)  /* SignalError "interval end precedes start"   energy.py:93-94 */
#define DW_E_SPAN (-2)      /* SignalError "interval [lo,hi] outside signal span [s,e]" energy.py:95-97 */
#define DW_E_EMPTY (-3)     /* SignalError "empty power signal"            energy.py:53 */
#define DW_E_ORDER (-4)     /* TraceError "power samples must be strictly increasing" trace_model.py:549-551 */
#define DW_E_ARG (-5)       /* bad argument (null/misaligned pointer, n < 0, threshold) */
#define DW_E_CUDA (-6)      /* a CUDA runtime error (launch failure, ...) */
#define DW_E_WORKSPACE (-7) /* workspace smaller than *_workspace_size() */
#define DW_E_UNSORTED (-8)  /* a set flagged sorted is not sorted by start */

/* --------------------------------------------------------------- constants */
#define DW_SIGNAL_STEP 0   /* ground truth: breakpoints of a piecewise-constant signal */
#define DW_SIGNAL_LINEAR 1 /* samples: trapezoid with linear interpolation */
#define DW_MAX_SETS 4      /* interval sets per dw_attribute call */
/* Intervals spanning at most DW_DIRECT_MAX segments are summed sequentially in
 * fp64 exactly as the reference does (bit-identical); longer ones are summed
 * exactly in 2^-40 W*us fixed point and rounded once. */
#ifndef DW_DIRECT_MAX
#define DW_DIRECT_MAX 256
#endif
/* How an interval's pieces are summed (dw_signal_t.sum_mode):
 *  DW_SUM_REFERENCE  the reference's sequential fp64 sum for intervals of at
 *                    most DW_DIRECT_MAX pieces (bit-identical to
 *                    energy.integrate), the exact sum below for longer ones;
 *  DW_SUM_EXACT      every interval as the exact sum of its pieces, each
 *                    rounded to 2^-40 W*us, rounded once to a double and
 *                    divided by 1e6.  Integer addition is associative, so the
 *                    result does not depend on how the device groups the
 *                    pieces (window prefixes, whole tiles); it differs from
 *                    the reference's sum by a few ulps.  Same
 *                    pieces, same values in both modes for every interval
 *                    longer than DW_DIRECT_MAX pieces and for the span total
 *                    of a signal with more than DW_DIRECT_MAX pieces. */
#define DW_SUM_REFERENCE 0
#define DW_SUM_EXACT 1
/* Tiling of the attribution kernel.  Whole tiles enter long-interval sums as
 * exact fixed-point tile sums (int128 sums of the rounded pieces), so any
 * grouping gives the oracle's value (oracle/dw_oracle.c fx_range). */
#ifndef DW_TILE
#define DW_TILE 1024
#endif
#ifndef DW_TILE_THREADS
#define DW_TILE_THREADS 192
#endif

/* ------------------------------------------------------------------- types */
typedef struct {
    const int64_t *d_ts;   /* [n] strictly increasing timestamps */
    const double *d_watts; /* [n] */
    int64_t n;
    int64_t span_hi; /* STEP: end of the last segment, max(trace end, ts[n-1]+1)
                        (energy.py:80); LINEAR: ignored, the span is [ts[0], ts[n-1]] */
    int32_t kind;    /* DW_SIGNAL_STEP | DW_SIGNAL_LINEAR */
    int32_t validate_order; /* 1: check ts strictly increasing (DW_E_ORDER) */
    int32_t sum_mode; /* DW_SUM_REFERENCE (0, default) | DW_SUM_EXACT (1) */
    int32_t pad;
} dw_signal_t;

typedef struct {
    const int64_t *d_start; /* [n] */
    const int64_t *d_end;   /* [n] */
    int64_t n;
    double *d_joules;       /* [n] out */
    int32_t sorted;         /* 1: d_start is non-decreasing (checked: DW_E_UNSORTED);
                               0: the library sorts a copy in the workspace */
    int32_t pad;
} dw_interval_set_t;

typedef struct {
    int32_t code;      /* first error class found, DW_OK if none */
    int32_t bad_set;   /* set of the reported interval, -1 if none */
    int64_t bad_index[DW_MAX_SETS]; /* per set: smallest index of an invalid interval, -1 if none */
    int64_t order_index;            /* first i with ts[i+1] <= ts[i], -1 if none */
    int64_t unsorted_index[DW_MAX_SETS]; /* first k with start[k] < start[k-1], -1 if none */
    int64_t long_intervals;         /* intervals that took the fixed-point path */
    double totals[4];               /* dw_ledger: total, operator_total, idle, unused */
} dw_status_t;

/* ---------------------------------------------------------- attribution */

/* Workspace bytes for dw_attribute / dw_ledger with these sizes. */
size_t dw_attribute_workspace_size(int64_t n_samples, const int64_t *set_sizes, int32_t nsets);

/* joules[k] = integral of the signal over [start[k], end[k]] for every set.
 * Replaces the per-interval energy.integrate calls of build_ledger
 * (energy.py:312-316).  Errors -> status (first invalid interval per set). */
int dw_attribute(const dw_signal_t *sig, dw_interval_set_t *sets, int32_t nsets,
                 void *d_workspace, size_t workspace_bytes, dw_stream_t stream);

/* build_ledger for one trace: sets[0] = operators, sets[1] = kernels (either may
 * be empty).  Also integrates the whole span and stores, in the status block,
 * totals = {total_joules, operator_total, idle_joules = max(total - op_total, 0)}
 * (energy.py:318-324).  operator_total is the exact sum rounded once. */
int dw_ledger(const dw_signal_t *sig, dw_interval_set_t *ops, dw_interval_set_t *kernels,
              void *d_workspace, size_t workspace_bytes, dw_stream_t stream);

/* One rank of a time-window-sharded trace.
 * The rank holds the samples [g_off, g_off + n) of a signal of
 * n_samples_global samples and owns the pieces (segments / trapezoid pieces,
 * indexed by their left sample) [piece_lo, piece_hi).  g_off must be a
 * multiple of DW_TILE, so the local tile grid is the global one. */
typedef struct {
    int64_t g_off, n_samples_global;
    int64_t piece_lo, piece_hi;
    int64_t ts_first, ts_last;  /* global first / last sample time (LINEAR edge rule) */
    double w_first, w_last;     /* and their watts */
} dw_window_t;

/* dw_attribute on the rank's local signal (sig: the local samples; for STEP,
 * span_hi = the next global sample time, or the global span end on the last
 * rank) for the intervals it computes whole, plus:
 *  - d_part[2e..2e+1]: exact int128 (2^-40 W*us, little-endian halves) share
 *    of listed interval e (d_blo/d_bhi, longer than DW_DIRECT_MAX pieces,
 *    crossing window edges) over the owned pieces -- summed over ranks and
 *    rounded once it equals the one-GPU value bit for bit;
 *  - d_tile_fx[2]: exact int128 sum of the owned whole-tile sums (the rank's
 *    share of the ledger total, same scale). */
int dw_attribute_window(const dw_signal_t *sig, dw_interval_set_t *sets, int32_t nsets, const dw_window_t *win,
                        const int64_t *d_blo, const int64_t *d_bhi, int64_t nb, int64_t *d_part,
                        int64_t *d_tile_fx, void *d_workspace, size_t workspace_bytes, dw_stream_t stream);

/* Cap the SMs the attribution tile kernel occupies (0 = all, the default), so
 * kernels on another stream can run beside it (pipeline.analyze overlaps the
 * join's pairing with the ledgers this way).  Process-wide. */
int dw_set_attribute_sms(int n);

/* Exact 2^-64 J fixed-point sum of d_x[0..n) as int128 halves (not rounded):
 * the per-rank share of a sharded operator_total.  Workspace as dw_fx_sum. */
int dw_fx_sum_exact(const double *d_x, int64_t n, int64_t *d_out_fx, void *d_workspace,
                    size_t workspace_bytes, dw_stream_t stream);

/* Overlap split (the north star's overlap-weighted
 * splitting for concurrent kernels, SURVEY.md G1 -- the reference has no such
 * mode: energy.py:305-316 gives every interval the full signal over its
 * span).  joules[k] for one set with the power divided equally among the
 * set's intervals active at each instant; equal to dw_attribute's result
 * whenever no two intervals of the set overlap.  Any order of intervals.
 * Errors as dw_attribute (status block at the head of the workspace, set 0). */
size_t dw_attribute_split_workspace_size(int64_t n_samples, int64_t n);
int dw_attribute_split(const dw_signal_t *sig, dw_interval_set_t *set, void *d_workspace,
                       size_t workspace_bytes, dw_stream_t stream);

/* Replay estimator (energy.py:196-256) for n_ops operators [start, end) of a
 * STEP ground truth: each op's power profile tiled `repeat` times, read by the
 * delayed sampler every period_us with the per-read delays d_delays (the
 * caller draws them: numpy PCG64 uniform(0.5, 1.5) x delay, the same stream
 * for every op, energy.py:160-165), mid-window reads averaged (Python sum()).
 * Out: d_watts[o] (steady power), d_joules[o] = watts * duration / 1e6.
 * *d_bad = first op whose profile is empty (the reference's SignalError),
 * INT64_MAX if none. */
int dw_replay(const dw_signal_t *truth, const int64_t *d_op_start, const int64_t *d_op_end, int64_t n_ops,
              int64_t repeat, int64_t period_us, const double *d_delays, int64_t n_delays, double *d_watts,
              double *d_joules, int64_t *d_bad, dw_stream_t stream);

/* Packed columns: a sorted int64 column stored
 * as base + uint32 deltas (d_delta[0] is 0 or the offset of the first value)
 * decodes to d_out[i] = base + sum(d_delta[0..i]); with d_dur, also
 * d_end[i] = d_out[i] + d_dur[i] (interval ends from durations). */
size_t dw_unpack_workspace_size(int64_t n);
int dw_unpack_deltas(const uint32_t *d_delta, int64_t n, int64_t base, int64_t *d_out, const uint32_t *d_dur,
                     int64_t *d_end, void *d_workspace, size_t workspace_bytes, dw_stream_t stream);
/* Same with narrow columns: deltas of delta_bytes = 1 (int8, value =
 * delta_bias + d[i]), 2 or 4 (unsigned, value = delta_bias + d[i]); durations
 * of dur_bytes = 2 or 4.  d[0] is ignored: the first value is `base`.  The
 * packer picks the narrowest width the column fits. */
int dw_unpack_deltas_w(const void *d_delta, int32_t delta_bytes, int64_t delta_bias, int64_t n, int64_t base,
                       int64_t *d_out, const void *d_dur, int32_t dur_bytes, int64_t *d_end, void *d_workspace,
                       size_t workspace_bytes, dw_stream_t stream);
/* Sorted timestamps from bit-packed deltas: field i (width bits, 1..32, at
 * bit i*width of the little-endian 32-bit words; one padding word after the
 * last) holds delta_i - bias; d_out[0] = base, d_out[i] = d_out[i-1] + bias +
 * field i.  A regular sampling clock with a few us of jitter packs its
 * timestamps into 1-4 bits each. */
int dw_unpack_bits(const uint32_t *d_words, int32_t width, int64_t bias, int64_t n, int64_t base, int64_t *d_out,
                   void *d_workspace, size_t workspace_bytes, dw_stream_t stream);
/* Timestamps of a clock with a nominal period (power meters polled at a
 * fixed rate, trace_model.py:63-65's power records), stored as residuals from
 * the linear predictor pred(i) = base + floor(i * step_fx / 2^32) (step_fx:
 * the period in 2^-32 us, < 2^63): field i (dw_unpack_bits layout; field 0
 * counts) holds ts[i] - pred(i) - bias, and d_out[i] = pred(i) + bias + field
 * i -- one independent decode per element (no scan).  A jittered clock's
 * residuals span half its deltas' range: one bit fewer per sample.  n < 2^31. */
int dw_unpack_grid(const uint32_t *d_words, int32_t width, int64_t bias, int64_t n, int64_t base, uint64_t step_fx,
                   int64_t *d_out, dw_stream_t stream);
/* Both in one pass: starts from bit-packed deltas as dw_unpack_bits, and
 * (d_dur_words non-NULL) d_end[i] = d_out[i] + dur_bias + duration field i,
 * as dw_unpack_bits_dur. */
int dw_unpack_bits_w(const uint32_t *d_words, int32_t width, int64_t bias, int64_t n, int64_t base, int64_t *d_out,
                     const uint32_t *d_dur_words, int32_t dur_width, int64_t dur_bias, int64_t *d_end,
                     void *d_workspace, size_t workspace_bytes, dw_stream_t stream);
/* Interval ends from bit-packed durations: d_end[i] = d_start[i] + bias +
 * field i (same field layout as dw_unpack_bits; field 0 counts). */
int dw_unpack_bits_dur(const int64_t *d_start, const uint32_t *d_words, int32_t width, int64_t bias, int64_t n,
                       int64_t *d_end, dw_stream_t stream);
/* Dictionary codes bit-packed (width bits each, dw_unpack_bits layout):
 * d_out[i] = d_dict[field i]. */
int dw_unpack_dict_bits(const uint64_t *d_dict, const uint32_t *d_words, int32_t width, int64_t n, uint64_t *d_out,
                        dw_stream_t stream);
/* Dictionary-coded 64-bit column (operator signatures): d_out[i] =
 * d_dict[code[i]], codes of code_bytes = 2 or 4. */
int dw_unpack_dict(const uint64_t *d_dict, const void *d_code, int32_t code_bytes, int64_t n, uint64_t *d_out,
                   dw_stream_t stream);
/* Watts stored as 9-significant-digit decimals (the trace format's on-disk
 * precision, trace_model.py:63-65): code = m | j << 30 (m < 2^30, j < 4),
 * d_out[i] = m * 10^-(p0 + j), one correctly rounded IEEE operation -- the
 * double a parse of the decimal text yields. */
int dw_unpack_decimal(const uint32_t *d_code, int64_t n, int32_t p0, double *d_out, dw_stream_t stream);

/* The same codes run-coded: a power meter read faster than it updates
 * repeats its last value, so only the samples that carry a new code store
 * one.  d_rep[(n + 31) / 32] is a bitmap, bit i % 32 of word i / 32 set when
 * sample i carries a new code (bit 0 must be set); d_code holds those codes in
 * sample order.  d_out[i] = the decoded code of the last new sample <= i. */
size_t dw_unpack_decimal_rep_workspace_size(int64_t n);
int dw_unpack_decimal_rep(const uint32_t *d_code, const uint32_t *d_rep, int64_t n, int32_t p0, double *d_out,
                          void *d_workspace, size_t workspace_bytes, dw_stream_t stream);
/* The same with the stored codes bit-packed: code k = bias + field k (width
 * bits, dw_unpack_bits layout; field 0 counts).  The packer strips the
 * decimal zeros every code shares (p0 lowered to match: integer-milliwatt
 * NVML readings keep ~20 bits) and packs the spread (C4: 30 instead of 32). */
int dw_unpack_decimal_rep_bits(const uint32_t *d_words, int32_t width, uint32_t bias, const uint32_t *d_rep, int64_t n,
                               int32_t p0, double *d_out, void *d_workspace, size_t workspace_bytes,
                               dw_stream_t stream);

/* JSONL ingestion (paper_2512_08365_b200/ingest.py):
 * byte-level stages over the raw file resident in HBM.  The canonical
 * power / op / kernel records of tensor-free traces parse here; `flags` (one
 * device unsigned) turns nonzero on anything else, and the caller then loads
 * the file through the reference-compatible Python loader.  Glue between the
 * stages (scans, compaction, sorts) is the caller's. */
int dw_ig_nl_count(const uint8_t *buf, int64_t n, unsigned long long *counts, unsigned *flags, dw_stream_t stream);
int dw_ig_nl_write(const uint8_t *buf, int64_t n, const unsigned long long *offs, int64_t *ends, dw_stream_t stream);
int dw_ig_classify(const uint8_t *buf, int64_t n, const int64_t *ends, int64_t nlines, uint8_t *type, unsigned *flags,
                   dw_stream_t stream);
int dw_ig_parse_power(const uint8_t *buf, const int64_t *ends, const int64_t *lines, int64_t m, int64_t *ts,
                      double *w, unsigned *flags, dw_stream_t stream);
/* tl_off / tl_len (may both be NULL): [2m] byte spans of each op's
 * input_tensor_ids and output_tensor_ids JSON lists (the host validates them
 * against the tensor records); NULL flags any tensor reference instead. */
int dw_ig_parse_op(const uint8_t *buf, const int64_t *ends, const int64_t *lines, int64_t m, int64_t *id_off,
                   int32_t *id_len, int64_t *name_off, int32_t *name_len, int64_t *kl_first, int32_t *kl_count,
                   int64_t *start, int64_t *end, int64_t *tl_off, int32_t *tl_len, unsigned *flags,
                   dw_stream_t stream);
int dw_ig_parse_kernel(const uint8_t *buf, const int64_t *ends, const int64_t *lines, int64_t m, int64_t *id_off,
                       int32_t *id_len, int64_t *name_off, int32_t *name_len, int64_t *corr, int64_t *start,
                       int64_t *end, unsigned *flags, dw_stream_t stream);
/* Word w (bytes 8w .. 8w+7) of each id span as a big-endian uint64, zero past
 * the id's end: sorting ids by these words, last word first (stable), gives
 * their byte-string order -- the op-id ranks of the report tie-break
 * (detect.py:265, nodes_a) computed at ingest. */
int dw_ig_id_words(const uint8_t *buf, const int64_t *off, const int32_t *len, int64_t m, int32_t w,
                   uint64_t *out, dw_stream_t stream);
int dw_ig_hash(const uint8_t *buf, const int64_t *off, const int32_t *len, int64_t m, uint64_t *h, uint32_t *idx,
               dw_stream_t stream);
int dw_ig_kernel_lists(const uint8_t *buf, int64_t nops, const int64_t *kl_first, const int32_t *kl_count,
                       const int64_t *kl_base, const int64_t *op_start, const int64_t *op_end, const uint64_t *kh,
                       const uint32_t *kidx, int64_t nk, const int64_t *k_off, const int32_t *k_len,
                       const int64_t *k_start, const int64_t *k_end, int64_t *fk_start, int64_t *fk_end,
                       int32_t *fk_op, int64_t *fk_kernel, unsigned *owner_count, unsigned *flags, dw_stream_t stream);

/* Synchronise `stream` and copy the status block out of the workspace. Returns
 * status->code. */
int dw_status(const void *d_workspace, dw_stream_t stream, dw_status_t *status);

/* The same read split in two, so a caller can queue more work before it
 * waits: dw_status_copy queues the copy of the workspace's DW_STATUS_BYTES
 * status block into h_block (pinned host memory; no synchronisation), and
 * dw_status_decode turns that copy -- once the stream has passed the copy --
 * into the status struct (same result and return code as dw_status). */
#define DW_STATUS_BYTES 256
int dw_status_copy(const void *d_workspace, void *h_block, dw_stream_t stream);
int dw_status_decode(const void *h_block, dw_status_t *status);

/* Exact (2^-64 J fixed point) sum of d_x[0..n) rounded once -> *d_out. */
size_t dw_fx_sum_workspace_size(int64_t n);
int dw_fx_sum(const double *d_x, int64_t n, double *d_out, void *d_workspace,
              size_t workspace_bytes, dw_stream_t stream);

/* PowerSignal.value_at for the sampler (energy.py:57-66, 160-171): watts of the
 * step signal at fractional times d_t (clamped to the span). */
int dw_step_value_at(const dw_signal_t *sig, const double *d_t, int64_t m, double *d_out,
                     dw_stream_t stream);

/* ------------------------------------------------------------------ diff */

/* Per-finding columns written by dw_detect_pairs / dw_join_diff.  Every column
 * but d_key_hi may be NULL (not written).  The ranking key is the 128-bit
 * (key_hi, key_lo), report order = descending: key_hi = waste flag << 63 |
 * bits of wasted_joules; key_lo = ~((tie + 1) << 32 | finding index) with tie
 * the rank of nodes_a.  When d_key_lo is NULL, dw_rank derives key_lo from the
 * join's numbering: tie = d_tie_rank[f] (or f when NULL) for f < n_a, -1 for
 * the B-only findings after them. */
typedef struct {
    double *d_energy_a, *d_energy_b; /* [P] */
    double *d_ratio;                 /* [P] high/low, 1.0 when equal, inf when low == 0 */
    int64_t *d_latency_a, *d_latency_b; /* [P] max end - min start */
    int8_t *d_verdict;               /* [P] 0 below_threshold, 1 tradeoff, 2 waste */
    int8_t *d_side;                  /* [P] 0 "-", 1 "A", 2 "B" */
    int8_t *d_informational;         /* [P] */
    double *d_wasted;                /* [P] high - low */
    uint64_t *d_key_hi, *d_key_lo;   /* [P] ranking key */
    const int64_t *d_tie_rank;       /* implicit key_lo: A-op id ranks (NULL = index) */
    int64_t n_a;                     /* implicit key_lo: number of A-op findings */
    /* the differential columns (north star (3)); each may be NULL */
    double *d_delta_e;               /* [P] e_b - e_a (J) */
    int64_t *d_delta_t;              /* [P] latency_b - latency_a (us) */
    double *d_epw_ratio;             /* [P] (e_b / work_b) / (e_a / work_a), IEEE (x/0 = inf, 0/0 = NaN);
                                        work = 1 per op without a work column */
} dw_findings_t;

/* detect_waste over CSR segment pairs (reference SubgraphPair lists).
 * Per pair p: members d_mem_a[d_off_a[p]..d_off_a[p+1]) index ops of trace A
 * (same for B).  Energies are CPython-3.12 sum() (Neumaier) over members in
 * order, as subgraph_joules does.  d_out_diff may be NULL (0.0).  d_tie[p] is
 * the rank of nodes_a under Python tuple order (the report tie-break). */
int dw_detect_pairs(int64_t P, const int64_t *d_off_a, const int32_t *d_mem_a,
                    const int64_t *d_off_b, const int32_t *d_mem_b,
                    const double *d_joules_a, const double *d_joules_b,
                    const int64_t *d_start_a, const int64_t *d_end_a,
                    const int64_t *d_start_b, const int64_t *d_end_b,
                    const double *d_out_diff, const int64_t *d_tie, double threshold,
                    dw_findings_t *out, dw_stream_t stream);

/* Order findings by (verdict != waste, -wasted_joules, nodes_a) -- detect.py:263-266.
 * Writes the k best finding indices, best first, into d_order (k <= P; k == P
 * is the full report order).  Also accumulates, into d_summary[0..3):
 * {n_waste, wasted_joules (exact sum over waste findings), n_findings}. */
size_t dw_rank_workspace_size(int64_t P, int64_t k);
int dw_rank(int64_t P, const dw_findings_t *f, int64_t k, int64_t *d_order, double *d_summary,
            void *d_workspace, size_t workspace_bytes, dw_stream_t stream);

/* Segmented top-k: the report order of many finding sets in one
 * call -- one segment per trace pair of a corpus (report() per pair,
 * detect.py:256-278).  Segment i's keys are as in dw_findings_t (d_key_lo NULL:
 * implied by the join numbering, d_tie_rank / n_a).  Writes, per segment, the
 * min(k, P_i) best finding indices into d_order[i * k ...] (rest -1), and
 * {n_waste, wasted_joules (exact), P_i, 0} into d_summary[4 * i ...] (may be
 * NULL).  k <= 8192. */
typedef struct {
    const uint64_t *d_key_hi, *d_key_lo;
    const int64_t *d_tie_rank;
    int64_t n_a;
    int64_t P;
} dw_rank_segment_t;
size_t dw_rank_segmented_workspace_size(int32_t nseg, int64_t k);
int dw_rank_segmented(const dw_rank_segment_t *segs, int32_t nseg, int64_t k, int64_t *d_order,
                      double *d_summary, void *d_workspace, size_t workspace_bytes, dw_stream_t stream);

/* The report rows of a join's top-k (d_order[k], join numbering) for the host:
 * d_out[6][k] int64 = A op, B op (-1 when empty), latency_a, latency_b, and
 * the joules of each side as f64 bits (0 when empty). */
int dw_topk_rows(const int64_t *d_order, int64_t k, int64_t n_a, const int32_t *d_match_a, const int32_t *d_b_only,
                 const double *d_joules_a, const double *d_joules_b, const int64_t *d_start_a,
                 const int64_t *d_end_a, const int64_t *d_start_b, const int64_t *d_end_b, int64_t *d_out,
                 dw_stream_t stream);

/* Signature hash-join diff.  Operators of A and B
 * are keyed by (sig, occurrence in op order); equal keys pair up, unmatched
 * operators become one-sided findings.  Findings are numbered: A ops in order
 * (f < n_a: matched or A-only), then B-only ops in B order (f = n_a + r).
 * Outputs: d_match_a[i] = B op paired with A op i or -1; d_b_only[r] = the
 * r-th B-only op; finding columns (out); d_epw_* (may be NULL) joules per unit
 * of useful work (d_work NULL = 1 per op).  d_rank (A side) is the
 * lexicographic rank of each A op id (report tie-break; NULL = index).
 * *d_count receives {P, n_matched, n_a_only, n_b_only}. */
typedef struct {
    const uint64_t *d_sig;   /* [n] */
    const int64_t *d_start, *d_end; /* [n] */
    const double *d_joules;  /* [n] attributed energy */
    const double *d_work;    /* [n] or NULL */
    const int64_t *d_rank;   /* [n] id rank (A side tie-break), NULL = index */
    int64_t n;
} dw_join_side_t;

/* max_distinct bounds the number of distinct signatures (hash table of
 * 2 x max_distinct slots; <= 0 means na + nb).  DW_E_WORKSPACE is returned if
 * the table overflows; retry with a larger bound.  Finding columns other than
 * the keys may be NULL (not written). */
size_t dw_join_workspace_size(int64_t na, int64_t nb, int64_t max_distinct);
int dw_join_diff(const dw_join_side_t *a, const dw_join_side_t *b, int64_t max_distinct,
                 double threshold, dw_findings_t *out, int32_t *d_match_a, int32_t *d_b_only,
                 double *d_epw_a, double *d_epw_b, int64_t *d_count, void *d_workspace,
                 size_t workspace_bytes, dw_stream_t stream);

/* dw_join_diff in two phases, so the pairing (signatures only) can run on its
 * own stream while the ledgers that provide the joules are still computing:
 * dw_join_prepare pairs the operators (d_match_a's sort state, d_b_only and
 * *n_b_only), dw_join_findings then writes the finding columns.  Both take
 * the same sides, max_distinct and workspace; the workspace carries the state
 * from one call to the other. */
int dw_join_prepare(const dw_join_side_t *a, const dw_join_side_t *b, int64_t max_distinct, int32_t *d_match_a,
                    int32_t *d_b_only, int64_t *n_b_only, void *d_workspace, size_t workspace_bytes,
                    dw_stream_t stream);
int dw_join_findings(const dw_join_side_t *a, const dw_join_side_t *b, int64_t max_distinct, double threshold,
                     dw_findings_t *out, int32_t *d_match_a, int32_t *d_b_only, int64_t n_b_only, double *d_epw_a,
                     double *d_epw_b, int64_t *d_count, void *d_workspace, size_t workspace_bytes,
                     dw_stream_t stream);

/* --------------------------------------------------------------- misc */
/* ---------------------------------------------- tensor equivalence (8(f)4)
 * Replaces the Python loops of subgraph_match.match_tensors
 * (subgraph_match.py:109-204) and tensor_equiv.singular_values /
 * invariant_set (tensor_equiv.py:118-189). */

/* norms[i] = sqrt(sum(v*v for v in values[off[i]:off[i+1]])) with CPython's
 * sum() -- the prefilter norms (subgraph_match.py:129-132), bit-exact. */
int dw_tensor_norms(const double *d_values, const int64_t *d_off, int64_t n, double *d_norms, dw_stream_t stream);

/* Prefilter (subgraph_match.py:134-145): (a, b) survives when count_a[a] ==
 * count_b[b] and, on every run r, |na - nb| <= eps * max(min(na, nb), 1e-30)
 * with na = d_norm_a[r * n_a + a].  pass 0 writes d_row_count[a]; pass 1,
 * given the exclusive scan d_row_off, writes the pairs in row-major order. */
int dw_tensor_prefilter(int pass, int64_t n_a, int64_t n_b, int32_t runs, const int64_t *d_count_a,
                        const int64_t *d_count_b, const double *d_norm_a, const double *d_norm_b, double eps,
                        int64_t *d_row_count, const int64_t *d_row_off, int64_t *d_pair_a, int64_t *d_pair_b,
                        dw_stream_t stream);

/* One unfolding of a row-major tensor: modes whose bit is set in `mask`
 * (ascending) index the rows, the others the columns (tensor_equiv.unfold). */
typedef struct {
    int64_t value_off;    /* first element of the tensor in d_values */
    int64_t out_off;      /* min(rows, cols) singular values written here */
    int64_t scratch_off;  /* rows*cols + min(rows, cols) doubles of d_scratch, used
                             when that exceeds smem_doubles */
    int32_t order;        /* 2..8 */
    int32_t mask;         /* proper, non-empty subset of the modes */
    int32_t dims[8];
} dw_unfold_t;

/* largest per-matrix working set (doubles) that fits in shared memory */
int64_t dw_unfold_smem_doubles(void);

/* Singular values of every unfolding by one-sided Jacobi with the reference's
 * round-robin order, tolerance and sweep cap (tensor_equiv.py:118-159):
 * sorted descending at d_spectra[out_off...]; d_spectra_len[i] = how many are
 * >= 1e-12.  smem_doubles = max over the batch of rows*cols + min(rows, cols),
 * capped at dw_unfold_smem_doubles(). */
int dw_unfold_spectra(const double *d_values, const dw_unfold_t *d_mats, int64_t n_mats, int64_t smem_doubles,
                      double *d_spectra, int32_t *d_spectra_len, double *d_scratch, dw_stream_t stream);

/* Bottleneck injective embedding (tensor_equiv.py:183-242) of spectrum set
 * job_a[j] against set job_b[j] (the smaller into the larger): set s is
 * unfoldings set_first[s] .. + set_count[s] (<= DW_EMBED_MAX_SPECTRA), unfolding
 * u is d_spec[u_off[u] .. + u_len[u]].  d_score[j] = the smallest level <= eps
 * admitting a perfect matching, +inf when none does. */
#define DW_EMBED_MAX_SPECTRA 14
int dw_spectra_embed(const double *d_spec, const int64_t *d_u_off, const int32_t *d_u_len, const int64_t *d_set_first,
                     const int32_t *d_set_count, int64_t n_jobs, const int64_t *d_job_a, const int64_t *d_job_b,
                     double eps, double *d_score, dw_stream_t stream);

/* ------------------------------------------- time-window join exchange (8(e))
 * Replaces shard.py's pack + sort-by-destination + NCCL all-to-all of the
 * sharded signature join (the reference has no multi-GPU path; SURVEY.md
 * 8(e)) with one kernel storing records straight into the receivers' buffers
 * through CUDA IPC mappings (P2P over NVLink/NVSwitch). */
#define DW_MAX_PEERS 64
#define DW_XCH_MAX_WIDTH 8
#define DW_IPC_HANDLE_BYTES 64

/* d_counts[d] = number of records (one per operator, d_sig[i]) bound for rank
 * d = ((sig ^ (sig >> 31)) & 0x7FFFFFFF) % world. */
int dw_exchange_count(const int64_t *d_sig, int64_t n, int32_t world, uint64_t *d_counts, dw_stream_t stream);
/* Record i (the width int64 columns cols[0..width-1] at row i) is stored at
 * d_peer[d] + (base[d] + slot) * width for its destination d, slot a
 * per-destination counter (d_cursor[world], reset here).  cols, d_peer and
 * base are HOST arrays of device pointers / offsets. */
int dw_exchange_scatter(const int64_t *const *cols, int32_t width, const int64_t *d_sig, int64_t n, int32_t world,
                        int64_t *const *d_peer, const int64_t *base, uint64_t *d_cursor, dw_stream_t stream);
/* Arrival flags of a persistent receive buffer: after its scatter, a sender
 * stores `epoch` into slot [me] of every receiver's flag array
 * (d_peer_flags[d]: receiver d's array, IPC-mapped; system-scope release after
 * a system fence); dw_exchange_wait holds the receiver's stream until every
 * sender's slot of d_flags[world] reaches `epoch` (device-side; *d_timeout
 * set to 1 if a sender never signals within ~20 s).  d_peer_flags is a HOST
 * array of device pointers. */
int dw_exchange_signal(uint64_t *const *d_peer_flags, int32_t world, int32_t me, uint64_t epoch,
                       dw_stream_t stream);
int dw_exchange_wait(const uint64_t *d_flags, int32_t world, uint64_t epoch, int32_t *d_timeout,
                     dw_stream_t stream);
/* CUDA IPC plumbing for the receive buffers (64-byte handles).  A buffer
 * inside a larger allocation exports the allocation's handle plus its byte
 * offset; the opener adds the offset to what dw_ipc_open returns. */
int dw_ipc_handle(const void *d_ptr, void *handle_out, int64_t *offset_out);
int dw_ipc_open(const void *handle, void **d_ptr_out);
int dw_ipc_close(void *d_ptr);

/* ------------------------------------------- misconfiguration probe (8(f)3)
 * Batched kernel-name alignment of analyze_segment_pair (diagnose.py:203-224):
 * per problem p, the token sequences a = d_tok_a[d_off_a[p] .. d_off_a[p+1])
 * and b (same for B) -- kernel names interned to integers -- are aligned on
 * their longest common subsequence with the reference's tie rule (on a
 * mismatch skip a's element when table[i+1][j] >= table[i][j+1]); matched
 * positions get flag 1 in d_match_a / d_match_b (indexed like the tokens).
 * d_tab: int32 scratch, problem p's (n+1)(m+1) table at d_tab_off[p]. */
int dw_lcs_matched(const int32_t *d_tok_a, const int64_t *d_off_a, const int32_t *d_tok_b, const int64_t *d_off_b,
                   int64_t nprob, const int64_t *d_tab_off, int32_t *d_tab, uint8_t *d_match_a, uint8_t *d_match_b,
                   dw_stream_t stream);

const char *dw_version(void);
const char *dw_error_string(int code);
/* number of kernel launches issued by this library on the calling thread
 * since the last reset (bench.py's gpu_launches) */
int64_t dw_launch_count(int reset);
/* Profiling hook for bench.py's roofline: when enabled, CUDA events bracket
 * every attribution tile-kernel launch on its stream; dw_kernel_time_ms
 * synchronises them and returns the summed device time, and
 * dw_kernel_timed_count the number of launches that time covers (every
 * launch: a full event ring is folded into the sum, never dropped). */
int dw_kernel_timing(int enable);
double dw_kernel_time_ms(int reset);
int64_t dw_kernel_timed_count(int reset);

#ifdef __cplusplus
}
#endif
#endif /* DWB200_H */
