// ingest.cu -- JSONL trace ingestion on the GPU.
//
// The reference parses a trace line by line with json.loads and builds
// frozen dataclasses (trace_model.py:341-492; O(N^2) duplicate-op test at
// :419).  Here the raw file bytes go to HBM once and every line is parsed by
// its own thread.  The fast path accepts exactly the canonical form that
// trace_to_lines writes (compact separators, fixed key order) for the three
// record types that carry the columns -- power, op, kernel -- on traces
// without tensor snapshots; every other line is handed back to the host.
// Anything unusual (another key order, escapes, a number the fast decimal
// conversion cannot round exactly, a semantic violation) makes the caller
// fall back to the reference-compatible Python loader, which then raises
// the reference's exact error.  So a trace either loads here with the same
// columns the Python path would build, or is loaded by the Python path.
//
// Steps (device): newline scan (block counts -> scan -> positions, plus a
// flag for bytes Python's splitlines() also treats as line breaks) ->
// classify every line -> per-type compaction -> per-type field parsing ->
// validation (power order, interval rules, unique ids / correlation ids by
// sorted 64-bit string hashes with byte comparison on equal hashes, kernel
// ownership and containment) -> the flattened kernel columns in op.kernel_ids
// order.
#include <cub/cub.cuh>

#include "dw_common.cuh"

namespace dw {

constexpr int IG_THREADS = 256;
constexpr int IG_BYTES = 256;  // bytes scanned per thread in the newline pass

enum : uint8_t { L_EMPTY = 0, L_POWER = 1, L_OP = 2, L_KERNEL = 3, L_OTHER = 4, L_BAD = 5 };

// flag bits (ingest status word)
enum : unsigned { F_ODD_BYTE = 1, F_BAD_LINE = 2, F_NUMBER = 4, F_ORDER = 8, F_INTERVAL = 16, F_DUP = 32,
                  F_OWNER = 64, F_TENSOR = 128, F_STRING = 256 };

__device__ __forceinline__ bool odd_byte(uint8_t c) {
    // splitlines() breaks at \r \v \f \x1c-\x1e (and non-ASCII separators); tabs are fine
    return c == '\r' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1e) || c >= 0x80 || (c < 0x20 && c != '\n' && c != '\t');
}

__global__ void nl_count_kernel(const uint8_t *buf, int64_t n, unsigned long long *counts, unsigned *flags) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t a = t * IG_BYTES;
    unsigned c = 0;
    bool odd = false;
    if (a < n) {
        const int64_t b = min(a + IG_BYTES, n);
        for (int64_t i = a; i < b; ++i) {
            const uint8_t x = buf[i];
            c += x == '\n';
            odd |= odd_byte(x);
        }
    }
    if (odd) atomicOr(flags, F_ODD_BYTE);
    counts[t] = c;
}

__global__ void nl_write_kernel(const uint8_t *buf, int64_t n, const unsigned long long *offs, int64_t *ends) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t a = t * IG_BYTES;
    if (a >= n) return;
    const int64_t b = min(a + IG_BYTES, n);
    unsigned long long o = offs[t];
    for (int64_t i = a; i < b; ++i)
        if (buf[i] == '\n') ends[o++] = i;
}

// ------------------------------------------------------------------ cursor
struct Cur {
    const uint8_t *p, *e;
    __device__ __forceinline__ bool lit(const char *s) {
        const uint8_t *q = p;
        for (; *s; ++s, ++q)
            if (q >= e || *q != (uint8_t)*s) return false;
        p = q;
        return true;
    }
    __device__ __forceinline__ bool at_end() const { return p == e; }
    // JSON integer (canonical: no leading zeros), fits int64
    __device__ bool int64v(int64_t &v) {
        bool neg = false;
        if (p < e && *p == '-') { neg = true; ++p; }
        if (p >= e || *p < '0' || *p > '9') return false;
        if (*p == '0' && p + 1 < e && p[1] >= '0' && p[1] <= '9') return false;
        uint64_t x = 0;
        int nd = 0;
        while (p < e && *p >= '0' && *p <= '9') {
            if (++nd > 18) return false;  // keep clear of overflow (Python would take it; we fall back)
            x = x * 10 + (*p++ - '0');
        }
        if (p < e && (*p == '.' || *p == 'e' || *p == 'E')) return false;  // not an integer literal
        v = neg ? -(int64_t)x : (int64_t)x;
        return true;
    }
    // JSON number -> the correctly rounded double (Clinger's fast path: at
    // most 15 significant digits and |decimal exponent| <= 22, where one IEEE
    // multiply or divide by an exact power of ten rounds correctly); false
    // when outside it (the caller falls back to Python's float()).
    __device__ bool number(double &v) {
        bool neg = false;
        if (p < e && *p == '-') { neg = true; ++p; }
        if (p >= e || *p < '0' || *p > '9') return false;
        if (*p == '0' && p + 1 < e && p[1] >= '0' && p[1] <= '9') return false;
        uint64_t m = 0;
        int nd = 0, e10 = 0;
        bool nz = false;
        while (p < e && *p >= '0' && *p <= '9') {
            const int d = *p++ - '0';
            if (nz || d) { nz = true; if (++nd > 15) return false; }
            m = m * 10 + d;
        }
        if (p < e && *p == '.') {
            ++p;
            if (p >= e || *p < '0' || *p > '9') return false;
            while (p < e && *p >= '0' && *p <= '9') {
                const int d = *p++ - '0';
                if (nz || d) { nz = true; if (++nd > 15) return false; }
                m = m * 10 + d;
                --e10;
            }
        }
        if (p < e && (*p == 'e' || *p == 'E')) {
            ++p;
            bool eneg = false;
            if (p < e && (*p == '+' || *p == '-')) { eneg = *p == '-'; ++p; }
            if (p >= e || *p < '0' || *p > '9') return false;
            int x = 0;
            while (p < e && *p >= '0' && *p <= '9') {
                x = x * 10 + (*p++ - '0');
                if (x > 400) return false;
            }
            e10 += eneg ? -x : x;
        }
        double r = (double)m;  // exact: m < 10^15 < 2^53
        if (m != 0) {
            if (e10 < -22 || e10 > 22) return false;
            double pw = 1.0;
            for (int i = 0; i < (e10 < 0 ? -e10 : e10); ++i) pw *= 10.0;  // exact for <= 22
            r = e10 < 0 ? __ddiv_rn(r, pw) : __dmul_rn(r, pw);
        }
        v = neg ? -r : r;
        return true;
    }
};

// span of a string at the cursor (absolute file offsets)
__device__ __forceinline__ bool take_str(Cur &c, const uint8_t *buf0, int64_t &off, int32_t &len) {
    if (c.p >= c.e || *c.p != '"') return false;
    const uint8_t *s = ++c.p;
    while (c.p < c.e && *c.p != '"') {
        if (*c.p == '\\') return false;
        ++c.p;
    }
    if (c.p >= c.e) return false;
    off = s - buf0;
    len = (int32_t)(c.p - s);
    ++c.p;
    return true;
}

// a list of strings "[...]"; count and span of the list body
__device__ __forceinline__ bool take_str_list(Cur &c, const uint8_t *buf0, int32_t &count, int64_t &first) {
    if (!c.lit("[")) return false;
    count = 0;
    first = c.p - buf0;
    if (c.lit("]")) return true;
    for (;;) {
        int64_t o;
        int32_t l;
        if (!take_str(c, buf0, o, l)) return false;
        ++count;
        if (c.lit("]")) return true;
        if (!c.lit(",")) return false;
    }
}

// skip one JSON value (for kernel params): objects, arrays, strings without
// escapes, numbers, true / false / null
__device__ bool skip_value(Cur &c, int depth) {
    if (c.p >= c.e || depth > 16) return false;
    const uint8_t x = *c.p;
    if (x == '{' || x == '[') {
        const uint8_t close = x == '{' ? '}' : ']';
        ++c.p;
        if (c.p < c.e && *c.p == close) { ++c.p; return true; }
        for (;;) {
            if (x == '{') {
                int64_t o; int32_t l;
                const uint8_t *b0 = c.p;
                if (!take_str(c, b0, o, l) || !c.lit(":")) return false;
            }
            if (!skip_value(c, depth + 1)) return false;
            if (c.p < c.e && *c.p == close) { ++c.p; return true; }
            if (!c.lit(",")) return false;
        }
    }
    if (x == '"') {
        int64_t o; int32_t l;
        return take_str(c, c.p, o, l);
    }
    if (c.lit("true") || c.lit("false") || c.lit("null")) return true;
    double d;
    return c.number(d);
}

__global__ void classify_kernel(const uint8_t *buf, int64_t n, const int64_t *ends, int64_t nlines, uint8_t *type,
                                unsigned *flags) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nlines) return;
    const int64_t a = i == 0 ? 0 : ends[i - 1] + 1;
    const int64_t b = ends[i];
    Cur c{buf + a, buf + b};
    // whitespace-only lines are skipped (raw.strip() is empty)
    bool blank = true;
    for (const uint8_t *q = c.p; q < c.e; ++q)
        if (*q != ' ' && *q != '\t') { blank = false; break; }
    uint8_t t;
    if (blank) t = L_EMPTY;
    else if (c.lit("{\"type\":\"power\",")) t = L_POWER;
    else if (c.lit("{\"type\":\"op\",")) t = L_OP;
    else if (c.lit("{\"type\":\"kernel\",")) t = L_KERNEL;
    else t = L_OTHER;  // header, config, tensor, progmodel, blocktrace: decoded on the host
    type[i] = t;
}

__global__ void parse_power_kernel(const uint8_t *buf, const int64_t *ends, const int64_t *lines, int64_t m,
                                   int64_t *ts, double *w, unsigned *flags) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m) return;
    const int64_t i = lines[k];
    const int64_t a = i == 0 ? 0 : ends[i - 1] + 1;
    Cur c{buf + a, buf + ends[i]};
    int64_t t = 0;
    double v = 0.0;
    bool ok = c.lit("{\"type\":\"power\",\"timestamp\":") && c.int64v(t) && c.lit(",\"watts\":");
    bool num = ok && c.number(v);
    ok = num && c.lit("}") && c.at_end();
    if (!ok) atomicOr(flags, ok || !num ? F_BAD_LINE | F_NUMBER : F_BAD_LINE);
    if (ok && v < 0.0) atomicOr(flags, F_INTERVAL);  // PowerSample.validate: negative watts
    ts[k] = t;
    w[k] = v;
}

__global__ void parse_op_kernel(const uint8_t *buf, const int64_t *ends, const int64_t *lines, int64_t m,
                                int64_t *id_off, int32_t *id_len, int64_t *name_off, int32_t *name_len,
                                int64_t *kl_first, int32_t *kl_count, int64_t *start, int64_t *end,
                                int64_t *tl_off, int32_t *tl_len, unsigned *flags) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m) return;
    const int64_t i = lines[k];
    const int64_t a = i == 0 ? 0 : ends[i - 1] + 1;
    Cur c{buf + a, buf + ends[i]};
    int64_t io = 0, no = 0, kf = 0, s = 0, e = 0, dummy;
    int32_t il = 0, nl = 0, kc = 0, nin = 0, nout = 0;
    const uint8_t *lin = nullptr, *lout = nullptr, *lend = nullptr;
    bool ok = c.lit("{\"type\":\"op\",\"op_id\":") && take_str(c, buf, io, il) && c.lit(",\"op_name\":") &&
              take_str(c, buf, no, nl) && c.lit(",\"input_tensor_ids\":") && (lin = c.p, true) &&
              take_str_list(c, buf, nin, dummy) && c.lit(",\"output_tensor_ids\":") && (lout = c.p, true) &&
              take_str_list(c, buf, nout, dummy) && (lend = c.p, true) &&
              c.lit(",\"kernel_ids\":") && take_str_list(c, buf, kc, kf) && c.lit(",\"start\":") && c.int64v(s) &&
              c.lit(",\"end\":") && c.int64v(e) && c.lit("}") && c.at_end();
    if (!ok) atomicOr(flags, F_BAD_LINE);
    // tensor references: without span outputs the Python path validates them;
    // with them the host checks them against the trace's tensor records
    if (ok && (nin || nout) && !tl_off) atomicOr(flags, F_TENSOR);
    if (tl_off) {  // the two lists' JSON text: [input list] then [output list], back to back
        tl_off[2 * k] = ok ? lin - buf : 0;
        tl_len[2 * k] = ok ? (int32_t)(lout - lin - (int)sizeof(",\"output_tensor_ids\":") + 1) : 0;
        tl_off[2 * k + 1] = ok ? lout - buf : 0;
        tl_len[2 * k + 1] = ok ? (int32_t)(lend - lout) : 0;
    }
    if (ok && e < s) atomicOr(flags, F_INTERVAL);          // OperatorEvent.validate
    id_off[k] = io; id_len[k] = il; name_off[k] = no; name_len[k] = nl;
    kl_first[k] = kf; kl_count[k] = kc; start[k] = s; end[k] = e;
}

__global__ void parse_kernel_kernel(const uint8_t *buf, const int64_t *ends, const int64_t *lines, int64_t m,
                                    int64_t *id_off, int32_t *id_len, int64_t *name_off, int32_t *name_len,
                                    int64_t *corr, int64_t *start, int64_t *end, unsigned *flags) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m) return;
    const int64_t i = lines[k];
    const int64_t a = i == 0 ? 0 : ends[i - 1] + 1;
    Cur c{buf + a, buf + ends[i]};
    int64_t io = 0, no = 0, cr = 0, s = 0, e = 0, bf;
    int32_t il = 0, nl = 0, bc = 0;
    bool ok = c.lit("{\"type\":\"kernel\",\"kernel_id\":") && take_str(c, buf, io, il) &&
              c.lit(",\"kernel_name\":") && take_str(c, buf, no, nl) && c.lit(",\"correlation_id\":") &&
              c.int64v(cr) && c.lit(",\"start\":") && c.int64v(s) && c.lit(",\"end\":") && c.int64v(e) &&
              c.lit(",\"backtrace\":") && take_str_list(c, buf, bc, bf);
    if (ok && c.lit(",\"params\":")) ok = c.p < c.e && *c.p == '{' && skip_value(c, 0);
    ok = ok && c.lit("}") && c.at_end();
    if (!ok) atomicOr(flags, F_BAD_LINE);
    if (ok && (e <= s || bc == 0)) atomicOr(flags, F_INTERVAL);  // KernelEvent.validate
    id_off[k] = io; id_len[k] = il; name_off[k] = no; name_len[k] = nl;
    corr[k] = cr; start[k] = s; end[k] = e;
}

// word w of each id as a big-endian 64-bit integer, zero padded past its end:
// unsigned order of the words, most significant first = byte-string order
__global__ void id_words_kernel(const uint8_t *buf, const int64_t *off, const int32_t *len, int64_t m, int w,
                                uint64_t *out) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m) return;
    const int32_t n = len[k];
    const uint8_t *s = buf + off[k];
    uint64_t v = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const int32_t i = 8 * w + b;
        v = (v << 8) | (i < n ? (uint64_t)s[i] : 0ULL);
    }
    out[k] = v;
}

// 64-bit FNV-1a of a byte string
__device__ __forceinline__ uint64_t fnv(const uint8_t *s, int32_t n) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (int32_t i = 0; i < n; ++i) h = (h ^ s[i]) * 0x100000001b3ULL;
    return h;
}

__global__ void hash_strings_kernel(const uint8_t *buf, const int64_t *off, const int32_t *len, int64_t m,
                                    uint64_t *h, uint32_t *idx) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m) return;
    h[k] = fnv(buf + off[k], len[k]);
    idx[k] = (uint32_t)k;
}

__device__ __forceinline__ bool same_str(const uint8_t *buf, int64_t oa, int32_t la, int64_t ob, int32_t lb) {
    if (la != lb) return false;
    for (int32_t i = 0; i < la; ++i)
        if (buf[oa + i] != buf[ob + i]) return false;
    return true;
}

// every kernel-id list entry of op o -> its kernel (binary search over the
// sorted kernel-id hashes + byte compare); flattened kernel columns in
// op.kernel_ids order; ownership counts
__global__ void kernel_lists_kernel(const uint8_t *buf, int64_t nops, const int64_t *kl_first,
                                    const int32_t *kl_count, const int64_t *kl_base, const int64_t *op_start,
                                    const int64_t *op_end, const uint64_t *kh, const uint32_t *kidx, int64_t nk,
                                    const int64_t *k_off, const int32_t *k_len, const int64_t *k_start,
                                    const int64_t *k_end, int64_t *fk_start, int64_t *fk_end, int32_t *fk_op,
                                    int64_t *fk_kernel, unsigned *owner_count, unsigned *flags) {
    const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (o >= nops) return;
    Cur c{buf + kl_first[o], buf + kl_first[o] + (1LL << 40)};
    const int32_t cnt = kl_count[o];
    int64_t e = kl_base[o];
    for (int32_t q = 0; q < cnt; ++q, ++e) {
        int64_t so;
        int32_t sl;
        if (q) c.lit(",");
        take_str(c, buf, so, sl);
        const uint64_t h = fnv(buf + so, sl);
        int64_t lo = 0, hi = nk;
        while (lo < hi) {
            const int64_t m = (lo + hi) >> 1;
            if (kh[m] < h) lo = m + 1; else hi = m;
        }
        int64_t found = -1;
        for (int64_t r = lo; r < nk && kh[r] == h; ++r)
            if (same_str(buf, so, sl, k_off[kidx[r]], k_len[kidx[r]])) { found = kidx[r]; break; }
        if (found < 0) {
            atomicOr(flags, F_OWNER);  // references a missing kernel
            fk_start[e] = fk_end[e] = 0;
            fk_op[e] = (int32_t)o;
            fk_kernel[e] = -1;
            continue;
        }
        atomicAdd(owner_count + found, 1u);
        const int64_t ks = k_start[found], ke = k_end[found];
        if (ks < op_start[o] || ke > op_end[o]) atomicOr(flags, F_OWNER);  // kernel outside its operator
        fk_start[e] = ks;
        fk_end[e] = ke;
        fk_op[e] = (int32_t)o;
        fk_kernel[e] = found;
    }
}

static unsigned ig_blocks(int64_t n) { return (unsigned)std::max<int64_t>(1, ceil_div(n, IG_THREADS)); }

}  // namespace dw

using namespace dw;

extern "C" {

#define IG_LAUNCH(kernel, n, ...)                                                               \
    do {                                                                                       \
        if ((n) > 0) kernel<<<ig_blocks(n), IG_THREADS, 0, (cudaStream_t)stream>>>(__VA_ARGS__); \
        count_launch();                                                                        \
        DW_CHECK_LAUNCH();                                                                     \
        return DW_OK;                                                                          \
    } while (0)

/* Byte-level stages of JSONL ingestion; the glue
 * (scans, compaction, sorts) is the caller's (ingest.py).  `flags` is one
 * device unsigned: nonzero after any stage = take the Python path. */
int dw_ig_nl_count(const uint8_t *buf, int64_t n, unsigned long long *counts, unsigned *flags, dw_stream_t stream) {
    IG_LAUNCH(nl_count_kernel, ceil_div(n, IG_BYTES), buf, n, counts, flags);
}
int dw_ig_nl_write(const uint8_t *buf, int64_t n, const unsigned long long *offs, int64_t *ends, dw_stream_t stream) {
    IG_LAUNCH(nl_write_kernel, ceil_div(n, IG_BYTES), buf, n, offs, ends);
}
int dw_ig_classify(const uint8_t *buf, int64_t n, const int64_t *ends, int64_t nlines, uint8_t *type, unsigned *flags,
                   dw_stream_t stream) {
    IG_LAUNCH(classify_kernel, nlines, buf, n, ends, nlines, type, flags);
}
int dw_ig_parse_power(const uint8_t *buf, const int64_t *ends, const int64_t *lines, int64_t m, int64_t *ts,
                      double *w, unsigned *flags, dw_stream_t stream) {
    IG_LAUNCH(parse_power_kernel, m, buf, ends, lines, m, ts, w, flags);
}
int dw_ig_parse_op(const uint8_t *buf, const int64_t *ends, const int64_t *lines, int64_t m, int64_t *id_off,
                   int32_t *id_len, int64_t *name_off, int32_t *name_len, int64_t *kl_first, int32_t *kl_count,
                   int64_t *start, int64_t *end, int64_t *tl_off, int32_t *tl_len, unsigned *flags,
                   dw_stream_t stream) {
    if ((tl_off == nullptr) != (tl_len == nullptr)) return DW_E_ARG;
    IG_LAUNCH(parse_op_kernel, m, buf, ends, lines, m, id_off, id_len, name_off, name_len, kl_first, kl_count, start,
              end, tl_off, tl_len, flags);
}
int dw_ig_parse_kernel(const uint8_t *buf, const int64_t *ends, const int64_t *lines, int64_t m, int64_t *id_off,
                       int32_t *id_len, int64_t *name_off, int32_t *name_len, int64_t *corr, int64_t *start,
                       int64_t *end, unsigned *flags, dw_stream_t stream) {
    IG_LAUNCH(parse_kernel_kernel, m, buf, ends, lines, m, id_off, id_len, name_off, name_len, corr, start, end,
              flags);
}
int dw_ig_id_words(const uint8_t *buf, const int64_t *off, const int32_t *len, int64_t m, int32_t w,
                   uint64_t *out, dw_stream_t stream) {
    if (w < 0) return DW_E_ARG;
    IG_LAUNCH(id_words_kernel, m, buf, off, len, m, w, out);
}
int dw_ig_hash(const uint8_t *buf, const int64_t *off, const int32_t *len, int64_t m, uint64_t *h, uint32_t *idx,
               dw_stream_t stream) {
    IG_LAUNCH(hash_strings_kernel, m, buf, off, len, m, h, idx);
}
int dw_ig_kernel_lists(const uint8_t *buf, int64_t nops, const int64_t *kl_first, const int32_t *kl_count,
                       const int64_t *kl_base, const int64_t *op_start, const int64_t *op_end, const uint64_t *kh,
                       const uint32_t *kidx, int64_t nk, const int64_t *k_off, const int32_t *k_len,
                       const int64_t *k_start, const int64_t *k_end, int64_t *fk_start, int64_t *fk_end,
                       int32_t *fk_op, int64_t *fk_kernel, unsigned *owner_count, unsigned *flags, dw_stream_t stream) {
    IG_LAUNCH(kernel_lists_kernel, nops, buf, nops, kl_first, kl_count, kl_base, op_start, op_end, kh, kidx, nk,
              k_off, k_len, k_start, k_end, fk_start, fk_end, fk_op, fk_kernel, owner_count, flags);
}

}  // extern "C"
