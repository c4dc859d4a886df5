/*
 * oracle.c -- CPU restatement of the reference's direct sparse convolution
 * hot path.  TEST INFRASTRUCTURE ONLY: this file is the parity checker for the
 * sm_100a engine in paper_2011_06295_b200/.  It is loaded by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg,
 * never by the product path.
 *
 * Parity is PINNED: tests/test_oracle_golden.py checks every routine here
 * against golden vectors produced by running the reference package itself
 * (tests/golden/make_golden.py, PYTHONPATH=/root/reference/pkg/src).
 *
 * What it restates (file:line relative to /root/reference/pkg/src/sparseconv):
 *   orc_conv_sparse_*   conv_sparse() engine.py:68-87 driving
 *                       conv_sparse_kernel() _kernels.py:53-85
 *                       (o = bias; o += v*x per nonzero in colidx order, the
 *                        product and the sum rounded separately: built with
 *                        -ffp-contract=off so no FMA is formed)
 *   orc_conv_direct_*   conv_direct_kernel() _kernels.py:17-50 (dense oracle)
 *   orc_pad_input_*     pad_input() shapes.py:98-105
 *   orc_build_csr       build_csr() csr.py:120-165 with the zero-promotion
 *                       rule of select_padding_zeros() csr.py:94-117
 *
 * The builder works on raw element bit patterns (2/4/8-byte floats) so that a
 * promoted -0.0 keeps its sign bit exactly like the numpy gather at csr.py:156.
 * It deliberately uses a different algorithm from the product builder
 * (two linear nearest-nonzero sweeps + a qsort on (distance, index)).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* helpers                                                                   */
/* ------------------------------------------------------------------------ */

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

static int is_zero_bits(const unsigned char* p, int esize) {
    /* IEEE zero test: +0.0 and -0.0 are zero, every other pattern (incl. NaN)
     * is a nonzero -- numpy's flatnonzero / count_nonzero semantics. */
    if (esize == 2) { uint16_t v; memcpy(&v, p, 2); return (v & 0x7fffu) == 0; }
    if (esize == 4) { uint32_t v; memcpy(&v, p, 4); return (v & 0x7fffffffu) == 0; }
    uint64_t v; memcpy(&v, p, 8); return (v & 0x7fffffffffffffffull) == 0;
}

/* ------------------------------------------------------------------------ */
/* padding  (shapes.py:98-105)                                               */
/* ------------------------------------------------------------------------ */

#define DEF_PAD(T, SUF)                                                         \
void orc_pad_input_##SUF(const T* x, T* xp, int n, int c, int h, int w, int p) \
{                                                                               \
    int hp = h + 2 * p, wp = w + 2 * p;                                         \
    memset(xp, 0, sizeof(T) * (size_t)n * c * hp * wp);                        \
    for (long long plane = 0; plane < (long long)n * c; ++plane)                \
        for (int y = 0; y < h; ++y)                                             \
            memcpy(xp + (plane * hp + y + p) * wp + p,                          \
                   x + (plane * h + y) * w, sizeof(T) * w);                     \
}
DEF_PAD(float, f32)
DEF_PAD(double, f64)

/* ------------------------------------------------------------------------ */
/* sparse conv  (engine.py:68-87 + _kernels.py:53-85)                        */
/* xf: (n_run, C*Hp*Wp) padded+flattened input, n_run % sb == 0              */
/* out: (n_run, K, E, F)                                                     */
/* ------------------------------------------------------------------------ */

#define DEF_SPARSE(T, SUF)                                                      \
void orc_conv_sparse_kernel_##SUF(const T* xf, long long row_len,               \
        const T* values, const int32_t* colidx, const int32_t* rowptr,          \
        const T* bias, T* out, int n_run, int k_out, int e_out, int f_out,      \
        int wp, int stride, int sb)                                             \
{                                                                               \
    long long nblocks = n_run / sb;                                             \
    long long units = nblocks * k_out;                                          \
    long long plane_out = (long long)e_out * f_out;                             \
    _Pragma("omp parallel for schedule(static)")                                \
    for (long long u = 0; u < units; ++u) {                                     \
        long long blk = u / k_out;                                              \
        int k = (int)(u % k_out);                                               \
        int t0 = rowptr[k], t1 = rowptr[k + 1];                                 \
        for (long long i = blk * sb; i < (blk + 1) * sb; ++i) {                 \
            const T* x = xf + i * row_len;                                      \
            T* o = out + (i * k_out + k) * plane_out;                           \
            for (long long q = 0; q < plane_out; ++q) o[q] = bias[k];           \
            for (int t = t0; t < t1; ++t) {                                     \
                T v = values[t];                                                \
                long long base = colidx[t];                                     \
                for (int e = 0; e < e_out; ++e) {                               \
                    const T* xr = x + base + (long long)e * stride * wp;        \
                    T* orow = o + (long long)e * f_out;                         \
                    if (stride == 1) { /* _kernels.py:80-82 contiguous axpy */  \
                        for (int f = 0; f < f_out; ++f) {                       \
                            T prod = v * xr[f];                                 \
                            orow[f] = orow[f] + prod;                           \
                        }                                                       \
                    } else {                                                    \
                        for (int f = 0; f < f_out; ++f) {                       \
                            T prod = v * xr[(long long)f * stride];             \
                            orow[f] = orow[f] + prod;                           \
                        }                                                       \
                    }                                                           \
                }                                                               \
            }                                                                   \
        }                                                                       \
    }                                                                           \
}
DEF_SPARSE(float, f32)
DEF_SPARSE(double, f64)

/* ------------------------------------------------------------------------ */
/* dense direct conv  (_kernels.py:17-50)  w: (K, C, R, S)                   */
/* ------------------------------------------------------------------------ */

#define DEF_DIRECT(T, SUF)                                                      \
void orc_conv_direct_kernel_##SUF(const T* xf, const T* w, const T* bias,      \
        T* out, int n, int k_out, int c_in, int r_k, int s_k, int e_out,        \
        int f_out, int hp, int wp, int stride)                                  \
{                                                                               \
    long long plane = (long long)hp * wp;                                       \
    long long row_len = plane * c_in;                                           \
    long long plane_out = (long long)e_out * f_out;                             \
    _Pragma("omp parallel for schedule(static)")                                \
    for (long long u = 0; u < (long long)n * k_out; ++u) {                      \
        long long i = u / k_out;                                                \
        int k = (int)(u % k_out);                                               \
        const T* x = xf + i * row_len;                                          \
        T* o = out + (i * k_out + k) * plane_out;                               \
        for (long long q = 0; q < plane_out; ++q) o[q] = bias[k];               \
        for (int c = 0; c < c_in; ++c)                                          \
            for (int r = 0; r < r_k; ++r)                                       \
                for (int s = 0; s < s_k; ++s) {                                 \
                    T v = w[(((long long)k * c_in + c) * r_k + r) * s_k + s];   \
                    long long base = c * plane + (long long)r * wp + s;         \
                    for (int e = 0; e < e_out; ++e)                             \
                        for (int f = 0; f < f_out; ++f) {                       \
                            T prod = v * x[base + (long long)e * stride * wp    \
                                           + (long long)f * stride];            \
                            o[e * f_out + f] = o[e * f_out + f] + prod;         \
                        }                                                       \
                }                                                               \
    }                                                                           \
}
DEF_DIRECT(float, f32)
DEF_DIRECT(double, f64)

/* ------------------------------------------------------------------------ */
/* CSR builder  (csr.py:80-165)                                              */
/* ------------------------------------------------------------------------ */

/* Per-channel nonzero counts (analyze_sparsity, csr.py:80-91). */
void orc_channel_nnz(const void* w, int esize, int k, long long vol,
                     long long* nnz_out) {
    const unsigned char* b = (const unsigned char*)w;
    for (int ch = 0; ch < k; ++ch) {
        long long cnt = 0;
        for (long long j = 0; j < vol; ++j)
            cnt += !is_zero_bits(b + ((long long)ch * vol + j) * esize, esize);
        nnz_out[ch] = cnt;
    }
}

/* select_padding_zeros (csr.py:94-117): choose `deficit` zero positions of a
 * flat channel ordered by (distance to nearest ORIGINAL nonzero, index);
 * with no nonzeros, the lowest-index zeros.  Output sorted ascending.
 * Returns 0, or -1 if deficit exceeds the number of zeros. */
typedef struct { long long d, j; } orc_key;
static int orc_key_cmp(const void* a, const void* b) {
    const orc_key* x = (const orc_key*)a; const orc_key* y = (const orc_key*)b;
    if (x->d != y->d) return x->d < y->d ? -1 : 1;
    return x->j < y->j ? -1 : (x->j > y->j);
}

int orc_select_padding_zeros(const void* flat, int esize, long long len,
                             long long deficit, long long* out) {
    const unsigned char* b = (const unsigned char*)flat;
    if (deficit == 0) return 0;
    if (len <= 0) return -1;
    long long nzeros = 0;
    for (long long j = 0; j < len; ++j) nzeros += is_zero_bits(b + j * esize, esize);
    if (deficit > nzeros) return -1;
    /* nearest nonzero to the left / right by two linear sweeps */
    const long long INF = (long long)1 << 62;
    long long* dl = (long long*)malloc(sizeof(long long) * len);
    long long last = -1;
    for (long long j = 0; j < len; ++j) {
        if (!is_zero_bits(b + j * esize, esize)) last = j;
        dl[j] = last < 0 ? INF : j - last;
    }
    orc_key* keys = (orc_key*)malloc(sizeof(orc_key) * (nzeros ? nzeros : 1));
    long long nk = 0; last = -1;
    for (long long j = len - 1; j >= 0; --j) {
        if (!is_zero_bits(b + j * esize, esize)) { last = j; continue; }
        long long dr = last < 0 ? INF : last - j;
        keys[nk].d = dl[j] < dr ? dl[j] : dr;   /* all-zero channel: every d = INF, */
        keys[nk].j = j;                          /* so the index decides          */
        ++nk;
    }
    qsort(keys, (size_t)nk, sizeof(orc_key), orc_key_cmp);
    char* taken = (char*)calloc((size_t)len, 1);
    for (long long q = 0; q < deficit; ++q) taken[keys[q].j] = 1;
    long long o = 0;
    for (long long j = 0; j < len; ++j) if (taken[j]) out[o++] = j;
    free(taken); free(keys); free(dl);
    return 0;
}

/* build_csr (csr.py:120-165).  Caller sizes values/colidx for
 * sum(counts) entries: pass nnz_cap; the function writes rowptr (k+1),
 * values (raw element bits), colidx (int32 padded-plane offsets) and returns
 * the stored entry count, or -1 on failure. */
long long orc_build_csr(const void* w, int esize, int k, int c, int r, int s,
                        int hp, int wp, int unify, long long nnz_cap,
                        void* values, int32_t* colidx, int32_t* rowptr,
                        int* level_out) {
    const unsigned char* b = (const unsigned char*)w;
    long long vol = (long long)c * r * s;
    long long* cnt = (long long*)malloc(sizeof(long long) * (k > 0 ? k : 1));
    orc_channel_nnz(w, esize, k, vol, cnt);
    long long target = 0;
    for (int ch = 0; ch < k; ++ch) if (cnt[ch] > target) target = cnt[ch];
    long long* pad = (long long*)malloc(sizeof(long long) * (vol > 0 ? vol : 1));
    char* keep = (char*)malloc((size_t)(vol > 0 ? vol : 1));
    long long pos = 0, maxcnt = 0;
    rowptr[0] = 0;
    for (int ch = 0; ch < k; ++ch) {
        const unsigned char* row = b + (long long)ch * vol * esize;
        for (long long j = 0; j < vol; ++j) keep[j] = !is_zero_bits(row + j * esize, esize);
        if (unify && cnt[ch] < target) {
            if (orc_select_padding_zeros(row, esize, vol, target - cnt[ch], pad) != 0) {
                free(cnt); free(pad); free(keep); return -1;
            }
            for (long long q = 0; q < target - cnt[ch]; ++q) keep[pad[q]] = 1;
        }
        long long here = 0;
        for (long long j = 0; j < vol; ++j) {
            if (!keep[j]) continue;
            if (pos >= nnz_cap) { free(cnt); free(pad); free(keep); return -1; }
            memcpy((unsigned char*)values + pos * esize, row + j * esize, esize);
            long long cc = j / ((long long)r * s);
            long long rem = j % ((long long)r * s);
            long long rr = rem / s, ss = rem % s;
            colidx[pos] = (int32_t)(cc * hp * wp + rr * wp + ss);
            ++pos; ++here;
        }
        if (here > maxcnt) maxcnt = here;
        rowptr[ch + 1] = (int32_t)pos;
    }
    *level_out = (int)(unify ? target : maxcnt);
    free(cnt); free(pad); free(keep);
    return pos;
}
