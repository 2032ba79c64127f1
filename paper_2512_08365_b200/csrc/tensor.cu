// tensor.cu -- tensor-equivalence prefilter and batched one-sided Jacobi SVD
// on B200 (sm_100a).
//
// The reference pairs tensors across two traces (subgraph_match.py:109-204):
// a cheap prefilter on element counts and Frobenius norms over every recorded
// run, then, per surviving pair, the multi-mode SVD invariant sets
// (tensor_equiv.py:118-189): the singular values of every non-trivial
// unfolding of each tensor, by one-sided Jacobi with a round-robin rotation
// order.  At config 1 that is ~125 s of Python.  Here:
//
//  K-norm   one thread per snapshot, CPython-3.12 sum() of v*v then sqrt --
//           bit-identical to the reference's prefilter norms;
//  K-pre    one CTA per A tensor scans all B tensors (counts equal, norm gap
//           within eps on every run); a count pass and an ordered write pass
//           give the candidates in np.nonzero (row-major) order;
//  K-svd    one CTA per unfolding: the unfolded matrix is gathered straight
//           from the tensor (mixed-radix index map, no host transpose) into
//           shared memory (global scratch when larger), taller than wide;
//           each sweep tests the reference's off-diagonal measure, then runs
//           the round-robin rounds with one warp per column pair (the pairs
//           of a round touch disjoint columns, so they rotate concurrently,
//           as the reference's vectorised round does); column norms are
//           ranked descending and trimmed at 1e-12.
//
// Floating point: the norms are exact; singular values agree with the
// reference's numpy Jacobi to rounding (dot products are summed in another
// order), the bar used by tests/test_gpu_tensor.py.
#include <cfloat>
#include <math_constants.h>

#include "dw_common.cuh"

namespace dw {

constexpr int TS_THREADS = 256;
constexpr int TS_WARPS = TS_THREADS / 32;
constexpr double JACOBI_TOL = 1e-14;   // tensor_equiv.py:26
constexpr int JACOBI_MAX_SWEEPS = 60;  // tensor_equiv.py:27
constexpr double SPECTRUM_FLOOR = 1e-12;
constexpr int SVD_SMEM_DOUBLES = 24 * 1024;  // 192 KB of matrix in shared memory

__global__ void tensor_norms_kernel(const double *values, const int64_t *off, int64_t n, double *out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    PySum s;
    for (int64_t k = off[i]; k < off[i + 1]; ++k) {
        const double v = values[k];
        s.add(__dmul_rn(v, v));
    }
    out[i] = __dsqrt_rn(s.result());
}

__device__ __forceinline__ bool pre_match(int64_t a, int64_t b, int64_t na, int64_t nb, int runs,
                                          const int64_t *count_a, const int64_t *count_b, const double *norm_a,
                                          const double *norm_b, double eps) {
    if (count_a[a] != count_b[b]) return false;
    for (int r = 0; r < runs; ++r) {
        const double x = norm_a[(int64_t)r * na + a], y = norm_b[(int64_t)r * nb + b];
        const double lo = fmin(x, y), diff = fabs(__dsub_rn(x, y));
        if (!(diff <= __dmul_rn(eps, fmax(lo, 1e-30)))) return false;  // subgraph_match.py:142-144
    }
    return true;
}

// pass 0: candidates per A row; pass 1: write them in column order
__global__ void tensor_prefilter_kernel(int pass, int64_t na, int64_t nb, int runs, const int64_t *count_a,
                                        const int64_t *count_b, const double *norm_a, const double *norm_b,
                                        double eps, int64_t *row_count, const int64_t *row_off, int64_t *pair_a,
                                        int64_t *pair_b) {
    __shared__ int64_t warp_tot[TS_WARPS];
    __shared__ int64_t base;
    const int64_t a = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) base = pass ? row_off[a] : 0;
    __syncthreads();
    for (int64_t b0 = 0; b0 < nb; b0 += TS_THREADS) {
        const int64_t b = b0 + threadIdx.x;
        const bool hit = b < nb && pre_match(a, b, na, nb, runs, count_a, count_b, norm_a, norm_b, eps);
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) warp_tot[w] = __popc(m);
        __syncthreads();
        int64_t before = 0, tot = 0;
        for (int k = 0; k < TS_WARPS; ++k) {
            before += k < w ? warp_tot[k] : 0;
            tot += warp_tot[k];
        }
        if (pass && hit) {
            const int64_t at = base + before + __popc(m & ((1u << lane) - 1u));
            pair_a[at] = a;
            pair_b[at] = b;
        }
        __syncthreads();
        if (threadIdx.x == 0) base += tot;
        __syncthreads();
    }
    if (!pass && threadIdx.x == 0) row_count[a] = base;
}

// ------------------------------------------------------------------ Jacobi
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// player at position pos of round rd (tensor_equiv.py:85-99: position 0 fixed,
// the rest rotated right once per round; n odd adds a bye = -1)
__device__ __forceinline__ int rr_player(int pos, int rd, int k, int n) {
    if (pos == 0) return 0;
    const int p = 1 + ((pos - 1 - rd) % (k - 1) + (k - 1)) % (k - 1);
    return p < n ? p : -1;
}

__global__ void __launch_bounds__(TS_THREADS) unfold_svd_kernel(const double *values, const dw_unfold_t *mats,
                                                                double *spectra, int32_t *spectra_len,
                                                                double *scratch, int64_t smem_doubles) {
    extern __shared__ double smem[];
    __shared__ double red[TS_WARPS];
    __shared__ int stop;
    const dw_unfold_t u = mats[blockIdx.x];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // the unfolding: modes in `mask` (ascending) index rows, the rest columns
    int64_t rows = 1, cols = 1;
    for (int d = 0; d < u.order; ++d) {
        if (u.mask >> d & 1) rows *= u.dims[d]; else cols *= u.dims[d];
    }
    const bool tr = cols > rows;  // work on the taller side (tensor_equiv.py:129-132)
    const int64_t M = tr ? cols : rows;
    const int N = (int)(tr ? rows : cols);
    // column-major, N columns of M, then N column norms
    double *A = M * N + N <= smem_doubles ? smem : scratch + u.scratch_off;
    const double *src = values + u.value_off;
    for (int64_t e = threadIdx.x; e < rows * cols; e += TS_THREADS) {
        // e = r * cols + c in the unfolded matrix; map (r, c) to the tensor offset
        int64_t r = e / cols, c = e - r * cols, off = 0, stride = 1;
        for (int d = u.order - 1; d >= 0; --d) {  // row-major tensor: last mode fastest
            int64_t idx;
            if (u.mask >> d & 1) { idx = r % u.dims[d]; r /= u.dims[d]; }
            else { idx = c % u.dims[d]; c /= u.dims[d]; }
            off += idx * stride;
            stride *= u.dims[d];
        }
        const int64_t ur = e / cols, uc = e - ur * cols;
        const int64_t i = tr ? uc : ur, j = tr ? ur : uc;  // row i, column j of the working matrix
        A[j * M + i] = src[off];
    }
    __syncthreads();
    if (N > 1) {
        const int k = N + (N & 1);
        for (int sweep = 0; sweep < JACOBI_MAX_SWEEPS; ++sweep) {
            // off-diagonal measure max |g_pq| / (d_p d_q) (tensor_equiv.py:102-110)
            double worst = 0.0;
            for (int64_t pq = w; pq < (int64_t)N * N; pq += TS_WARPS) {
                const int p = (int)(pq / N), q = (int)(pq - (int64_t)p * N);
                if (q <= p) continue;
                double g = 0.0, dp = 0.0, dq = 0.0;
                for (int64_t i = lane; i < M; i += 32) {
                    const double x = A[(int64_t)p * M + i], y = A[(int64_t)q * M + i];
                    g = __fma_rn(x, y, g);
                    dp = __fma_rn(x, x, dp);
                    dq = __fma_rn(y, y, dq);
                }
                g = warp_sum(g);
                dp = warp_sum(dp);
                dq = warp_sum(dq);
                const double den = __dmul_rn(sqrt(fmax(dp, 0.0)), sqrt(fmax(dq, 0.0)));
                double ratio = fabs(g) / den;
                if (isnan(ratio)) ratio = 0.0;
                if (isinf(ratio)) ratio = DBL_MAX;
                worst = fmax(worst, ratio);
            }
            if (lane == 0) red[w] = worst;
            __syncthreads();
            if (threadIdx.x == 0) {
                double m = 0.0;
                for (int i = 0; i < TS_WARPS; ++i) m = fmax(m, red[i]);
                stop = m <= JACOBI_TOL;
            }
            __syncthreads();
            if (stop) break;
            for (int rd = 0; rd < k - 1; ++rd) {
                for (int i = w; i < k / 2; i += TS_WARPS) {
                    int p = rr_player(i, rd, k, N), q = rr_player(k - 1 - i, rd, k, N);
                    if (p < 0 || q < 0) continue;
                    if (p > q) { const int t = p; p = q; q = t; }
                    double *cp = A + (int64_t)p * M, *cq = A + (int64_t)q * M;
                    double al = 0.0, be = 0.0, ga = 0.0;
                    for (int64_t r = lane; r < M; r += 32) {
                        const double x = cp[r], y = cq[r];
                        al = __fma_rn(x, x, al);
                        be = __fma_rn(y, y, be);
                        ga = __fma_rn(x, y, ga);
                    }
                    al = warp_sum(al);
                    be = warp_sum(be);
                    ga = warp_sum(ga);
                    const double scale = sqrt(fmax(al * be, 0.0));
                    if (!(fabs(ga) > JACOBI_TOL * (scale > 0.0 ? scale : 1.0))) continue;
                    const double zeta = (be - al) / (2.0 * ga);
                    double t = zeta == 0.0 ? 1.0 : copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                    const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
                    for (int64_t r = lane; r < M; r += 32) {
                        const double x = cp[r], y = cq[r];
                        cp[r] = x * c - y * s;
                        cq[r] = x * s + y * c;
                    }
                }
                __syncthreads();
            }
        }
    }
    // column norms, ranked descending (ties by column), trimmed at the floor
    double *nrm = A + (int64_t)N * M;
    for (int j = w; j < N; j += TS_WARPS) {
        double s = 0.0;
        for (int64_t r = lane; r < M; r += 32) s = __fma_rn(A[(int64_t)j * M + r], A[(int64_t)j * M + r], s);
        s = warp_sum(s);
        if (lane == 0) nrm[j] = sqrt(s);
    }
    __syncthreads();
    __shared__ int kept;
    if (threadIdx.x == 0) kept = 0;
    __syncthreads();
    for (int j = threadIdx.x; j < N; j += TS_THREADS) {
        const double v = nrm[j];
        int rank = 0;
        for (int i = 0; i < N; ++i) {
            const double o = nrm[i];
            rank += (o > v) || (o == v && i < j);
        }
        spectra[u.out_off + rank] = v;
        if (v >= SPECTRUM_FLOOR) atomicAdd(&kept, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) spectra_len[blockIdx.x] = kept;
}


// ------------------------------------------------- bottleneck embedding
// tensor_equiv.py:183-242 for one (small set, large set) job per thread:
// distances with the reference's sequential arithmetic (diff summed in index
// order, norms by CPython sum()), the levels <= eps sorted, Kuhn augmenting
// paths on bitmask rows, binary search for the smallest feasible level.
constexpr int EMBED_MAX = DW_EMBED_MAX_SPECTRA;

struct Kuhn {
    uint32_t adj[EMBED_MAX];
    int owner[EMBED_MAX];
    int rows, cols;
    // augmenting path from row `root` (iterative DFS: no recursion, so the
    // stack frame is static)
    __device__ bool augment(int root, uint32_t &seen) {
        int row[EMBED_MAX], via[EMBED_MAX];
        uint32_t cand[EMBED_MAX];
        int depth = 0;
        row[0] = root;
        cand[0] = adj[root];
        while (depth >= 0) {
            const uint32_t c = cand[depth] & ~seen;
            if (!c) { --depth; continue; }
            const int j = __ffs(c) - 1;
            cand[depth] = c & (c - 1);
            seen |= 1u << j;
            via[depth] = j;
            if (owner[j] < 0) {
                for (int d = depth; d >= 0; --d) owner[via[d]] = row[d];
                return true;
            }
            ++depth;
            row[depth] = owner[j];
            cand[depth] = adj[owner[j]];
        }
        return false;
    }
    __device__ bool perfect(const double *d, double limit) {
        for (int i = 0; i < rows; ++i) {
            uint32_t m = 0;
            for (int j = 0; j < cols; ++j) m |= (d[i * EMBED_MAX + j] <= limit ? 1u : 0u) << j;
            adj[i] = m;
        }
        for (int j = 0; j < cols; ++j) owner[j] = -1;
        for (int i = 0; i < rows; ++i) {
            uint32_t seen = 0;
            if (!augment(i, seen)) return false;
        }
        return true;
    }
};

__device__ double spec_norm(const double *s, int n) {
    PySum acc;
    for (int i = 0; i < n; ++i) acc.add(__dmul_rn(s[i], s[i]));
    return __dsqrt_rn(acc.result());
}

__global__ void spectra_embed_kernel(const double *spec, const int64_t *u_off, const int32_t *u_len,
                                     const int64_t *set_first, const int32_t *set_count, int64_t n_jobs,
                                     const int64_t *job_a, const int64_t *job_b, double eps, double *score) {
    const int64_t jb = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (jb >= n_jobs) return;
    int64_t sa = job_a[jb], sb = job_b[jb];
    if (set_count[sa] > set_count[sb]) { const int64_t t = sa; sa = sb; sb = t; }  // small into large
    const int rows = set_count[sa], cols = set_count[sb];
    if (rows == 0) { score[jb] = 0.0; return; }
    double d[EMBED_MAX * EMBED_MAX], lv[EMBED_MAX * EMBED_MAX];
    double nl[EMBED_MAX];
    for (int j = 0; j < cols; ++j) {
        const int64_t u = set_first[sb] + j;
        nl[j] = spec_norm(spec + u_off[u], u_len[u]);
    }
    int nlv = 0;
    for (int i = 0; i < rows; ++i) {
        const int64_t ui = set_first[sa] + i;
        const double *x = spec + u_off[ui];
        const int lx = u_len[ui];
        const double nx = spec_norm(x, lx);
        for (int j = 0; j < cols; ++j) {
            const int64_t uj = set_first[sb] + j;
            const double *y = spec + u_off[uj];
            const int ly = u_len[uj], n = lx > ly ? lx : ly;
            double dist = 0.0;
            if (n) {
                double diff = 0.0;
                for (int k = 0; k < n; ++k) {
                    const double t = __dsub_rn(k < lx ? x[k] : 0.0, k < ly ? y[k] : 0.0);
                    diff = __dadd_rn(diff, __dmul_rn(t, t));
                }
                dist = __ddiv_rn(__dsqrt_rn(diff), fmax(fmin(nx, nl[j]), 1e-30));
            }
            d[i * EMBED_MAX + j] = dist;
            if (dist <= eps) {  // insert into the sorted unique level list
                int k = nlv;
                while (k > 0 && lv[k - 1] > dist) --k;
                if (!(k > 0 && lv[k - 1] == dist)) {
                    for (int m = nlv; m > k; --m) lv[m] = lv[m - 1];
                    lv[k] = dist;
                    ++nlv;
                }
            }
        }
    }
    Kuhn km;
    km.rows = rows;
    km.cols = cols;
    if (nlv == 0 || !km.perfect(d, lv[nlv - 1])) { score[jb] = CUDART_INF; return; }
    int lo = 0, hi = nlv - 1;
    while (lo < hi) {
        const int mid = (lo + hi) / 2;
        if (km.perfect(d, lv[mid])) hi = mid; else lo = mid + 1;
    }
    score[jb] = lv[lo];
}

}  // namespace dw

using namespace dw;

extern "C" {

int dw_tensor_norms(const double *d_values, const int64_t *d_off, int64_t n, double *d_norms, dw_stream_t stream) {
    if (n < 0 || (n && (!d_values || !d_off || !d_norms))) return DW_E_ARG;
    if (n) {
        tensor_norms_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, (cudaStream_t)stream>>>(d_values, d_off, n,
                                                                                         d_norms);
        count_launch();
    }
    DW_CHECK_LAUNCH();
    return DW_OK;
}

int dw_tensor_prefilter(int pass, int64_t n_a, int64_t n_b, int32_t runs, const int64_t *d_count_a,
                        const int64_t *d_count_b, const double *d_norm_a, const double *d_norm_b, double eps,
                        int64_t *d_row_count, const int64_t *d_row_off, int64_t *d_pair_a, int64_t *d_pair_b,
                        dw_stream_t stream) {
    if (n_a < 0 || n_b < 0 || runs < 0 || (pass != 0 && pass != 1)) return DW_E_ARG;
    if (pass == 0 && n_a && !d_row_count) return DW_E_ARG;
    if (pass == 1 && n_a && (!d_row_off || !d_pair_a || !d_pair_b)) return DW_E_ARG;
    if (n_a && n_b) {
        tensor_prefilter_kernel<<<(unsigned)n_a, TS_THREADS, 0, (cudaStream_t)stream>>>(
            pass, n_a, n_b, runs, d_count_a, d_count_b, d_norm_a, d_norm_b, eps, d_row_count, d_row_off, d_pair_a,
            d_pair_b);
        count_launch();
    } else if (pass == 0 && n_a) {
        cudaMemsetAsync(d_row_count, 0, n_a * sizeof(int64_t), (cudaStream_t)stream);
    }
    DW_CHECK_LAUNCH();
    return DW_OK;
}

int64_t dw_unfold_smem_doubles(void) { return SVD_SMEM_DOUBLES; }

int dw_unfold_spectra(const double *d_values, const dw_unfold_t *d_mats, int64_t n_mats, int64_t smem_doubles,
                      double *d_spectra, int32_t *d_spectra_len, double *d_scratch, dw_stream_t stream) {
    if (n_mats < 0 || smem_doubles < 0 || smem_doubles > SVD_SMEM_DOUBLES ||
        (n_mats && (!d_values || !d_mats || !d_spectra || !d_spectra_len)))
        return DW_E_ARG;
    if (n_mats) {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(unfold_svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 SVD_SMEM_DOUBLES * (int)sizeof(double));
            attr = true;
        }
        unfold_svd_kernel<<<(unsigned)n_mats, TS_THREADS, (size_t)smem_doubles * sizeof(double),
                            (cudaStream_t)stream>>>(d_values, d_mats, d_spectra, d_spectra_len, d_scratch,
                                                    smem_doubles);
        count_launch();
    }
    DW_CHECK_LAUNCH();
    return DW_OK;
}

int dw_spectra_embed(const double *d_spec, const int64_t *d_u_off, const int32_t *d_u_len, const int64_t *d_set_first,
                     const int32_t *d_set_count, int64_t n_jobs, const int64_t *d_job_a, const int64_t *d_job_b,
                     double eps, double *d_score, dw_stream_t stream) {
    if (n_jobs < 0 || (n_jobs && (!d_spec || !d_u_off || !d_u_len || !d_set_first || !d_set_count || !d_job_a ||
                                  !d_job_b || !d_score)))
        return DW_E_ARG;
    if (n_jobs) {
        spectra_embed_kernel<<<(unsigned)ceil_div(n_jobs, 64), 64, 0, (cudaStream_t)stream>>>(
            d_spec, d_u_off, d_u_len, d_set_first, d_set_count, n_jobs, d_job_a, d_job_b, eps, d_score);
        count_launch();
    }
    DW_CHECK_LAUNCH();
    return DW_OK;
}

}  // extern "C"
