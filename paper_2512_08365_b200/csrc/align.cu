// align.cu -- batched kernel-name alignment of the misconfiguration probe
// (diagnose.py:203-224 _lcs_matched, called per waste finding by
// analyze_segment_pair).  The reference aligns the two segments' kernel-name
// sequences with a longest-common-subsequence table and walks it with a fixed
// tie rule: on a mismatch, skip a's element when that does not shorten the
// remaining LCS (table[i+1][j] >= table[i][j+1]), else skip b's.  Here every
// finding's alignment is one thread (the sequences are a segment's kernels:
// short), names interned to integer tokens on the host, the suffix-LCS table
// in a caller workspace slice, the matched positions written as flags.
#include "dw_common.cuh"

namespace dw {

__global__ void lcs_matched_kernel(const int32_t *ta, const int64_t *off_a, const int32_t *tb, const int64_t *off_b,
                                   int64_t nprob, const int64_t *tab_off, int32_t *tab, uint8_t *match_a,
                                   uint8_t *match_b) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= nprob) return;
    const int32_t *a = ta + off_a[p], *b = tb + off_b[p];
    const int n = (int)(off_a[p + 1] - off_a[p]), m = (int)(off_b[p + 1] - off_b[p]);
    int32_t *T = tab + tab_off[p];  // (n + 1) x (m + 1), row-major: T[i * (m + 1) + j] = LCS(a[i:], b[j:])
    const int W = m + 1;
    for (int j = 0; j <= m; ++j) T[n * W + j] = 0;
    for (int i = n - 1; i >= 0; --i) {
        T[i * W + m] = 0;
        const int32_t ai = a[i];
        for (int j = m - 1; j >= 0; --j) {
            const int32_t down = T[(i + 1) * W + j], right = T[i * W + j + 1];
            T[i * W + j] = ai == b[j] ? 1 + T[(i + 1) * W + j + 1] : (down >= right ? down : right);
        }
    }
    uint8_t *ma = match_a + off_a[p], *mb = match_b + off_b[p];
    for (int i = 0; i < n; ++i) ma[i] = 0;
    for (int j = 0; j < m; ++j) mb[j] = 0;
    int i = 0, j = 0;
    while (i < n && j < m) {
        if (a[i] == b[j]) {
            ma[i] = 1;
            mb[j] = 1;
            ++i;
            ++j;
        } else if (T[(i + 1) * W + j] >= T[i * W + j + 1]) {
            ++i;
        } else {
            ++j;
        }
    }
}

}  // namespace dw

using namespace dw;

extern "C" {

int dw_lcs_matched(const int32_t *d_tok_a, const int64_t *d_off_a, const int32_t *d_tok_b, const int64_t *d_off_b,
                   int64_t nprob, const int64_t *d_tab_off, int32_t *d_tab, uint8_t *d_match_a, uint8_t *d_match_b,
                   dw_stream_t stream) {
    if (nprob < 0 || (nprob && (!d_off_a || !d_off_b || !d_tab_off || !d_tab || !d_match_a || !d_match_b)))
        return DW_E_ARG;
    if (nprob) {
        lcs_matched_kernel<<<(unsigned)ceil_div(nprob, 128), 128, 0, (cudaStream_t)stream>>>(
            d_tok_a, d_off_a, d_tok_b, d_off_b, nprob, d_tab_off, d_tab, d_match_a, d_match_b);
        count_launch();
    }
    DW_CHECK_LAUNCH();
    return DW_OK;
}

}  // extern "C"
